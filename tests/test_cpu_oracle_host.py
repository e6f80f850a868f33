"""CPU suite: the oracle pinned to the reference's golden outputs, the host
logic of the drop-in, and the C-ABI library surface (no compute calls)."""

import ctypes
import hashlib
import os
import re

import numpy as np
import pytest

from golden_inputs import CASES_ATTN, CASES_SCORE, SCORE_POLICIES, make_qkv

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def oracle():
    import oracle as o
    o.lib()
    return o


# ----------------------------- oracle pin ---------------------------------

@pytest.mark.parametrize("case", CASES_SCORE, ids=[c["name"] for c in CASES_SCORE])
def test_oracle_scoring_matches_reference_golden(oracle, case):
    z = np.load(os.path.join(GOLDEN, f"score_{case['name']}.npz"))
    q, k, _ = make_qkv(case["heads"], case["frames"] * (case["patches"] + case["specials"]),
                       case["d"], case["seed"])
    pidx = oracle.patch_indices(case["frames"], case["patches"], case["specials"])
    qp = oracle.block_pool(q[:, pidx], case["block_q"])
    kp = oracle.block_pool(k[:, pidx], case["block_k"])
    assert sha(qp) == str(z["qp_sha"])
    assert sha(kp) == str(z["kp_sha"])
    pr = oracle.pooled_scores(qp, kp, case["d"])
    if case["name"] in ("cfg1", "n100h2"):
        # large pooled GEMMs: OpenBLAS's sequential-FMA kernel, bit-exact
        assert sha(pr) == str(z["probs_sha"])
    else:
        # tiny GEMMs take OpenBLAS's small-matrix kernel (different FMA
        # order): probabilities agree to a few ulp, masks still exact
        np.testing.assert_allclose(pr[0, :16], z["probs_head0"], rtol=1e-5, atol=1e-7)
    nk = kp.shape[1]
    for i, (tau, rho) in enumerate(SCORE_POLICIES):
        m, _ = oracle.select_blocks(pr, tau, oracle.min_blocks(nk, rho))
        assert np.array_equal(oracle.pack_bits(m), z[f"mask{i}_bits"]), (tau, rho)


@pytest.mark.parametrize("case", CASES_ATTN[:3], ids=[c["name"] for c in CASES_ATTN[:3]])
def test_oracle_attention_matches_reference_golden(oracle, case):
    z = np.load(os.path.join(GOLDEN, f"attn_{case['name']}.npz"))
    F, P, S = case["frames"], case["patches"], case["specials"]
    q, k, v = make_qkv(case["heads"], F * (P + S), case["d"], case["seed"])
    pidx = oracle.patch_indices(F, P, S)
    m, _ = oracle.predict_mask(q[:, pidx], k[:, pidx], case["block_q"], case["block_k"],
                               case["tau"], case["rho"])
    assert np.array_equal(oracle.pack_bits(m), z["mask_bits"])
    port = oracle.sparse_attention_port(q, k, v, F, P, S, m, case["block_q"], case["block_k"],
                                        threads=2)
    assert np.array_equal(port, z["out"])  # fp32 port is bit-identical
    f64 = oracle.masked_attention_f64(q, k, v, F, P, S, m, case["block_q"], case["block_k"])
    assert np.abs(f64 - z["out"]).max() <= 1e-5


def test_oracle_exp_matches_numpy_on_avx512_hosts(oracle):
    flags = open("/proc/cpuinfo").read() if os.path.exists("/proc/cpuinfo") else ""
    if "avx512f" not in flags:
        pytest.skip("numpy's AVX512F exp is the pinned model")
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.uniform(-20, 0, 20000), rng.uniform(-103, -80, 2000),
                        -np.arange(0, 2000) * 1e-4]).astype(np.float32)
    assert np.array_equal(oracle.np_expf(x), np.exp(x))


def test_oracle_pairwise_matches_numpy_sum(oracle):
    rng = np.random.default_rng(1)
    for n in (1, 5, 8, 9, 127, 128, 129, 1000, 4279, 21391):
        a = rng.random(n).astype(np.float32)
        got = oracle.lib().oracle_pairwise_sum(a.ctypes.data_as(ctypes.c_void_p), n)
        assert np.float32(got) == np.float32(0.0) + a.sum(dtype=np.float32) or \
            np.float32(got) == a.sum(dtype=np.float32)


def test_oracle_live_against_reference(oracle, reference_pkg):
    """Only in the build container: the restatement vs the reference itself
    on a fresh seed (re-pins the numpy/OpenBLAS order model on this host)."""
    from bsattn.maskpred import block_pool, pooled_scores, select_blocks, MaskPolicy
    from bsattn.layout import BlockGeometry
    rng = np.random.default_rng(12345)
    q = rng.standard_normal((2, 9000, 64)).astype(np.float32)
    k = rng.standard_normal((2, 9000, 64)).astype(np.float32)
    qp, kp = block_pool(q, 128), block_pool(k, 64)
    assert np.array_equal(qp, oracle.block_pool(q, 128))
    assert np.array_equal(kp, oracle.block_pool(k, 64))
    pr = pooled_scores(qp, kp, 64)
    assert np.array_equal(pr, oracle.pooled_scores(qp, kp, 64))
    g = BlockGeometry(9000, 128, 64)
    for tau, rho in SCORE_POLICIES:
        ref = select_blocks(pr, MaskPolicy(tau, rho, g)).blocks
        got, _ = oracle.select_blocks(pr, tau, oracle.min_blocks(g.nk_blocks, rho))
        assert np.array_equal(ref, got)


# ----------------------------- host logic ---------------------------------

def test_layout_parity_with_reference_semantics():
    from paper_2509_07120_b200 import layout as L
    lay = L.TokenLayout(frames=2, patches_per_frame=2, specials_per_frame=1)
    perm, inv = L.partition_permutation(lay)
    assert perm.tolist() == [0, 3, 1, 2, 4, 5]
    assert np.array_equal(perm[inv], np.arange(6))
    g = L.BlockGeometry(257, 128, 64)
    assert (g.nq_blocks, g.nk_blocks) == (3, 5)
    assert g.q_block_sizes().tolist() == [128, 128, 1]
    assert g.k_block_sizes().tolist() == [64, 64, 64, 64, 1]
    vggt = L.TokenLayout(10, 1369, 5)
    assert L.attention_entry_count(vggt, patch_only=True) == 187_416_100
    assert L.attention_entry_count(vggt) == 13740 ** 2
    assert vggt.patch_grid == (37, 37)
    for idx in (0, 4, 5, 1373, 1374, 1379, 13739):
        f, kind, r, c = L.token_coords(vggt, idx)
        assert L.token_index(vggt, f, kind, r if kind == L.PATCH else idx % 1374, c) == idx
    late = L.TokenLayout(2, 3, 2, specials_first=False)
    assert L.partition_permutation(late)[0].tolist() == [3, 4, 8, 9, 0, 1, 2, 5, 6, 7]
    with pytest.raises(ValueError):
        L.TokenLayout(0, 5)
    with pytest.raises(ValueError):
        L.BlockGeometry(10, 0, 4)
    with pytest.raises(IndexError):
        L.token_coords(vggt, 13740)


def test_layout_matches_reference_package(reference_pkg):
    from paper_2509_07120_b200 import layout as L
    for f, p, s, sf in ((3, 90, 5, True), (2, 7, 0, True), (4, 13, 3, False)):
        ours = L.partition_permutation(L.TokenLayout(f, p, s, specials_first=sf))
        ref = reference_pkg.partition_permutation(reference_pkg.TokenLayout(f, p, s, specials_first=sf))
        assert all(np.array_equal(a, b) for a, b in zip(ours, ref))


def test_policy_min_blocks():
    from paper_2509_07120_b200.layout import BlockGeometry
    from paper_2509_07120_b200.maskpred import MaskPolicy
    assert MaskPolicy(0.0, 0.9, BlockGeometry(100, 1, 1)).min_blocks == 10
    assert MaskPolicy(0.0, 1.0, BlockGeometry(100, 1, 1)).min_blocks == 1
    assert MaskPolicy(0.0, 0.0, BlockGeometry(100, 1, 1)).min_blocks == 100
    assert MaskPolicy(0.0, 0.75, BlockGeometry(273800, 128, 64)).min_blocks == 1069
    for bad in (-0.1, 1.5):
        with pytest.raises(ValueError):
            MaskPolicy(bad, 0.5, BlockGeometry(10, 1, 1))
        with pytest.raises(ValueError):
            MaskPolicy(0.5, bad, BlockGeometry(10, 1, 1))


def test_bsm_roundtrip_host(tmp_path):
    from paper_2509_07120_b200.layout import BlockGeometry
    from paper_2509_07120_b200.maskpred import BlockMask, read_mask, write_mask
    rng = np.random.default_rng(0)
    g = BlockGeometry(1000, 128, 64)
    blocks = rng.random((3, g.nq_blocks, g.nk_blocks)) < 0.3
    blocks[:, :, 0] = True
    m = BlockMask(blocks, g)
    p = tmp_path / "m.bsm"
    write_mask(p, m)
    raw = p.read_bytes()
    assert raw[:4] == b"BSMK" and len(raw) == 16 + 3 * g.nq_blocks * 2
    assert np.array_equal(read_mask(p, g).blocks, blocks)
    with pytest.raises(ValueError, match="magic"):
        (tmp_path / "bad.bsm").write_bytes(b"XXXX" + raw[4:])
        read_mask(tmp_path / "bad.bsm", g)
    with pytest.raises(ValueError, match="size"):
        (tmp_path / "short.bsm").write_bytes(raw[:-1])
        read_mask(tmp_path / "short.bsm", g)
    empty = blocks.copy()
    empty[0, 1] = False
    with pytest.raises(ValueError, match="at least one"):
        BlockMask(empty, g)


def test_bsm_reads_reference_written_file(tmp_path, reference_pkg):
    from paper_2509_07120_b200.layout import BlockGeometry
    from paper_2509_07120_b200.maskpred import read_mask
    rng = np.random.default_rng(3)
    g = reference_pkg.BlockGeometry(700, 128, 64)
    blocks = rng.random((2, g.nq_blocks, g.nk_blocks)) < 0.5
    blocks[:, :, 3] = True
    reference_pkg.write_mask(tmp_path / "r.bsm", reference_pkg.BlockMask(blocks, g))
    assert np.array_equal(read_mask(tmp_path / "r.bsm", BlockGeometry(700, 128, 64)).blocks, blocks)


# ----------------------------- C ABI surface -------------------------------

def test_library_loads_and_exports_header_symbols():
    from paper_2509_07120_b200 import _native as N
    lib = ctypes.CDLL(N.LIB_PATH)
    header = open(os.path.join(ROOT, "include", "bsa.h")).read()
    declared = set(re.findall(r"\b(bsa_[a-z0-9_]+)\s*\(", header))
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(lib, name), f"libbsa.so does not export {name}"
    assert set(N.exported_symbols()) == declared
    L = N.lib()
    assert L.bsa_version() >= 100


def test_library_is_sm100a_only():
    from paper_2509_07120_b200 import _native as N
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches


def test_tensor_core_kernel_uses_tcgen05_and_tma():
    from paper_2509_07120_b200 import _native as N
    import subprocess
    out = subprocess.run(["cuobjdump", "-sass", N.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    for mnemonic in ("UTCHMMA", "UTMALDG", "LDTM", "STTM"):
        assert mnemonic in out.stdout, mnemonic
    # the fused QKV projection and output projection:
    # tcgen05 MMAs, TMA loads (multicast B halves) and TMA bulk tensor stores
    funcs = re.split(r"\n\s*Function : ", out.stdout)
    qkv = [f for f in funcs if f.split("\n", 1)[0].find("qkv_pool_kernel") >= 0]
    # pair / single-CTA x QKV projection / output projection + residual
    assert len(qkv) == 4, "four instances of qkv_pool_kernel"
    for body in qkv:
        for mnemonic in ("UTCHMMA", "UTMALDG", "UTMASTG", "LDTM"):
            assert mnemonic in body, mnemonic


def test_path_selection_without_gpu():
    from paper_2509_07120_b200 import _native as N
    L = N.lib()
    lay = N.BsaLayout(200, 1369, 5, 1)
    assert L.bsa_sparse_attention_path(lay, 64, 128, 64, N.BSA_BF16, 0) == N.PATH_TC
    assert L.bsa_sparse_attention_path(lay, 64, 128, 64, N.BSA_F32, 0) == N.PATH_TC  # X3
    assert L.bsa_sparse_attention_path(lay, 64, 128, 64, N.BSA_F32, 1) == N.PATH_SIMT
    assert L.bsa_sparse_attention_path(lay, 32, 64, 32, N.BSA_BF16, 0) == N.PATH_SIMT
    assert L.bsa_sparse_attention_path(lay, 32, 64, 32, N.BSA_BF16, 2) < 0
    ws = L.bsa_sparse_attention_workspace(lay, 16, 64, 128, 64, N.BSA_BF16, 0, 0)
    assert ws >= 3 * 16 * 274800 * 64 * 2


def test_synth_restatement_matches_reference_digests():
    """tests/golden_inputs.py's restatement of the reference's planted-match
    generator (synth.py:149-202) reproduces the reference's q/k/v bit for bit
    (digests written by make_golden.py from the reference itself)."""
    import hashlib

    from golden_inputs import c6_inputs

    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "c6_scene.npz"))
    for x, key in zip(c6_inputs(), ("q_sha", "k_sha", "v_sha")):
        assert hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest() == str(z[key])


def test_c6_masks_oracle_vs_reference(oracle):
    """The C restatement of the scoring stage gives the reference's C6 masks."""
    from golden_inputs import C6_RHOS, c6_inputs

    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "c6_scene.npz"))
    q, k, _ = c6_inputs()
    for i, rho in enumerate(C6_RHOS):
        m, _ = oracle.predict_mask(q, k, 128, 64, 0.0, rho)
        assert np.array_equal(oracle.pack_bits(m).reshape(z[f"mask{i}_bits"].shape),
                              z[f"mask{i}_bits"])
    m, _ = oracle.predict_mask(q, k, 128, 64, 0.9, 0.5)
    assert np.array_equal(oracle.pack_bits(m).reshape(z["cdf_bits"].shape), z["cdf_bits"])
