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
