"""The reference CLI flows (tests/test_cli.py:44-112 of the reference) run
unchanged through the B200 CLI: .bsat in, .bsm / .bsat out, same CSVs.
The mask file is compared byte-for-byte with the oracle's reference-order
mask."""

import csv
import io

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

COMMON = ["--frames", "2", "--patches-per-frame", "128", "--specials-per-frame", "0",
          "--block-q", "64", "--block-k", "32"]


@pytest.fixture
def scene(tmp_path):
    from paper_2509_07120_b200.tensorio import write_tensor
    rng = np.random.default_rng(1)
    for name in "qkv":
        write_tensor(tmp_path / f"s_{name}.bsat",
                     rng.standard_normal((1, 256, 32)).astype(np.float32))
    return tmp_path / "s"


def _run_csv(capsys, argv):
    from paper_2509_07120_b200.cli import main
    main(argv)
    return list(csv.reader(io.StringIO(capsys.readouterr().out)))


def test_sparse_pipeline_matches_dense_on_full_mask(tmp_path, scene):
    from paper_2509_07120_b200.cli import main
    from paper_2509_07120_b200.tensorio import read_tensor
    m, o_s, o_d = tmp_path / "m.bsm", tmp_path / "os.bsat", tmp_path / "od.bsat"
    main(["mask", "--q", f"{scene}_q.bsat", "--k", f"{scene}_k.bsat", "--tau", "0", "--rho", "0",
          "--out", str(m)] + COMMON)
    main(["attend", "--mode", "sparse", "--q", f"{scene}_q.bsat", "--k", f"{scene}_k.bsat",
          "--v", f"{scene}_v.bsat", "--mask", str(m), "--out", str(o_s)] + COMMON)
    main(["attend", "--mode", "dense", "--q", f"{scene}_q.bsat", "--k", f"{scene}_k.bsat",
          "--v", f"{scene}_v.bsat", "--out", str(o_d)])
    np.testing.assert_allclose(read_tensor(o_s), read_tensor(o_d), atol=1e-5)


def test_mask_file_matches_oracle(tmp_path, scene):
    import oracle
    from paper_2509_07120_b200.cli import main
    from paper_2509_07120_b200.tensorio import read_tensor
    m = tmp_path / "m.bsm"
    main(["mask", "--q", f"{scene}_q.bsat", "--k", f"{scene}_k.bsat", "--tau", "0.6",
          "--rho", "0.5", "--out", str(m)] + COMMON)
    q, k = read_tensor(f"{scene}_q.bsat"), read_tensor(f"{scene}_k.bsat")
    ref, _ = oracle.predict_mask(q, k, 64, 32, 0.6, 0.5)
    assert m.read_bytes()[16:] == oracle.pack_bits(ref).tobytes()


def test_mask_stats_csv(tmp_path, scene, capsys):
    rows = _run_csv(capsys, ["mask", "--q", f"{scene}_q.bsat", "--k", f"{scene}_k.bsat",
                             "--tau", "0", "--rho", "0.75", "--out", str(tmp_path / "m.bsm"),
                             "--stats"] + COMMON)
    assert rows[0] == ["head", "achieved_sparsity"]
    assert float(rows[1][1]) == pytest.approx(0.75, abs=0.01)


def test_attend_report_csv(tmp_path, scene, capsys):
    from paper_2509_07120_b200.cli import main
    m, out = tmp_path / "m.bsm", tmp_path / "o.bsat"
    main(["mask", "--q", f"{scene}_q.bsat", "--k", f"{scene}_k.bsat", "--tau", "0", "--rho",
          "0.5", "--out", str(m)] + COMMON)
    rows = _run_csv(capsys, ["attend", "--mode", "sparse", "--q", f"{scene}_q.bsat",
                             "--k", f"{scene}_k.bsat", "--v", f"{scene}_v.bsat", "--mask", str(m),
                             "--out", str(out), "--report"] + COMMON)
    assert rows[0] == ["head", "achieved_sparsity", "sparse_flops", "theoretical_speedup",
                       "wall_ms"]
    assert float(rows[1][1]) == pytest.approx(0.5, abs=0.01)
    assert out.exists()


def test_determinism_across_cli_runs(tmp_path, scene):
    from paper_2509_07120_b200.cli import main
    outs = []
    for tag in "xy":
        m, o = tmp_path / f"{tag}.bsm", tmp_path / f"{tag}.bsat"
        main(["mask", "--q", f"{scene}_q.bsat", "--k", f"{scene}_k.bsat", "--tau", "0.6",
              "--rho", "0.5", "--out", str(m)] + COMMON)
        main(["attend", "--mode", "sparse", "--q", f"{scene}_q.bsat", "--k", f"{scene}_k.bsat",
              "--v", f"{scene}_v.bsat", "--mask", str(m), "--out", str(o)] + COMMON)
        outs.append((m.read_bytes(), o.read_bytes()))
    assert outs[0] == outs[1]


def test_bench_csv_schema(tmp_path, capsys):
    rows = _run_csv(capsys, ["bench", "--sizes", "2048,4096", "--tau", "0", "--rho", "0.75",
                             "--repeats", "3", "--with-predict"])
    assert rows[0] == ["N", "dense_ms", "sparse_ms", "achieved_sparsity", "speedup", "predict_ms"]
    assert [int(r[0]) for r in rows[1:]] == [2048, 4096]
    assert all(float(r[3]) == pytest.approx(0.75, abs=0.02) for r in rows[1:])


def _write_map(tmp_path, n=16, heads=2, seed=0):
    """A post-softmax map as the reference's CLI test builds it (test_cli.py:114-123)."""
    from paper_2509_07120_b200.tensorio import write_tensor
    rng = np.random.default_rng(seed)
    logits = rng.standard_normal((heads, n, n)).astype(np.float32)
    m = np.exp(logits)
    m /= m.sum(axis=2, keepdims=True)
    path = tmp_path / "map.bsat"
    write_tensor(path, m)
    return path


def test_analyze_csv(tmp_path, capsys):
    """test_cli.py:125-136 of the reference."""
    path = _write_map(tmp_path)
    rows = _run_csv(capsys, ["analyze", "--map", str(path), "--frames", "2",
                             "--patches-per-frame", "6", "--specials-per-frame", "2",
                             "--layer", "15"])
    assert rows[0] == ["layer", "head", "quadrant", "mean", "max"]
    assert {r[2] for r in rows[1:]} == {"S2S", "S2P", "P2S", "P2P"}
    assert {r[1] for r in rows[1:]} == {"0", "1", "mean", "std"}
    assert all(r[0] == "15" for r in rows[1:])


def test_analyze_to_file(tmp_path):
    """test_cli.py:138-144 of the reference."""
    from paper_2509_07120_b200.cli import main
    path = _write_map(tmp_path)
    out = tmp_path / "stats.csv"
    main(["analyze", "--map", str(path), "--frames", "2", "--patches-per-frame", "6",
          "--specials-per-frame", "2", "--csv", str(out)])
    assert out.read_text().startswith("layer,head,quadrant")


def test_analyze_streamed_matches_map(tmp_path, capsys):
    """analyze --q/--k (no map) reports what analyze --map reports for the
    map of the same bf16 q/k."""
    import torch
    from paper_2509_07120_b200.tensorio import write_tensor
    rng = np.random.default_rng(5)
    H, F, P, S = 2, 3, 200, 5
    T = F * (P + S)
    q, k = (rng.standard_normal((H, T, 64)).astype(np.float32) for _ in range(2))
    q, k = (torch.from_numpy(x).to(torch.bfloat16).float().numpy() for x in (q, k))
    write_tensor(tmp_path / "q.bsat", q)
    write_tensor(tmp_path / "k.bsat", k)
    s = q.astype(np.float64) @ k.astype(np.float64).transpose(0, 2, 1) * np.float32(0.125)
    p = np.exp(s - s.max(axis=2, keepdims=True))
    p /= p.sum(axis=2, keepdims=True)
    write_tensor(tmp_path / "map.bsat", p.astype(np.float32))
    lay = ["--frames", str(F), "--specials-per-frame", str(S)]
    a = _run_csv(capsys, ["analyze", "--map", str(tmp_path / "map.bsat")] + lay)
    b = _run_csv(capsys, ["analyze", "--q", str(tmp_path / "q.bsat"), "--k",
                          str(tmp_path / "k.bsat")] + lay)
    assert [r[:3] for r in a] == [r[:3] for r in b]
    for ra, rb in zip(a[1:], b[1:]):
        if ra[1] == "std":
            continue  # std of 2 near-equal heads: relative tolerance is meaningless
        np.testing.assert_allclose([float(x) for x in rb[3:]], [float(x) for x in ra[3:]],
                                   rtol=5e-4)
