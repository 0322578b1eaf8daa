"""The callers either side of the hot path: the known-spectrum generator
(reference synthetic.py:63-112) and the randomized-vs-direct timing harness
(reference bench.py:72-136) on the device path, against outputs of the
reference itself (tests/golden/ref_synth.npz, made by make_synth_golden.py).
The reference's own tests for these are test_synthetic.py / test_bench.py:
determinism per seed, spectrum recovered by the direct method, record
fields and the seed rule."""
import dataclasses
import os

import numpy as np
import pytest

import paper_2404_09459_b200 as rg
from paper_2404_09459_b200 import bench as hb
from paper_2404_09459_b200 import cli

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "ref_synth.npz"))


def _host(dm):
    return dm.t.cpu().numpy()


@pytest.mark.parametrize("i", range(len(GOLD["cases"])))
def test_synth_gmp_matches_reference(i):
    m, p, n, frac, seed = GOLD["cases"][i]
    spec = rg.SynthSpec(m=int(m), p=int(p), n=int(n), rank_frac=float(frac), seed=int(seed),
                        field="real")
    res = rg.synth_gmp(spec)
    # the spectrum is pure RNG arithmetic: bit-identical
    assert np.array_equal(res.true_spectrum.alphas, GOLD[f"alphas_{i}"])
    assert np.array_equal(res.true_spectrum.betas, GOLD[f"betas_{i}"])
    assert [res.true_spectrum.r, res.true_spectrum.s] == list(GOLD[f"rs_{i}"])
    # the matrices go through this package's QR / GEMM kernels: rounding-level
    # agreement with LAPACK's (1e-12 of the matrix norm)
    for got, ref in ((_host(res.pair.g1), GOLD[f"g1_{i}"]), (_host(res.pair.g2), GOLD[f"g2_{i}"])):
        assert got.shape == ref.shape
        assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
    assert abs(res.condition_r - float(GOLD[f"cond_{i}"])) <= 1e-9 * float(GOLD[f"cond_{i}"])


def test_synth_deterministic_and_seed_sensitive():
    spec = rg.SynthSpec(m=30, p=25, n=10, rank_frac=0.8, seed=5, field="real")
    a, b = rg.synth_gmp(spec), rg.synth_gmp(spec)
    assert np.array_equal(_host(a.pair.g1), _host(b.pair.g1))
    assert np.array_equal(_host(a.pair.g2), _host(b.pair.g2))
    c = rg.synth_gmp(dataclasses.replace(spec, seed=6))
    assert not np.array_equal(_host(a.pair.g1), _host(c.pair.g1))


def test_direct_method_recovers_true_spectrum():
    """The generator's purpose (test_synthetic.py): the direct GSV of the
    pair is the prescribed spectrum, up to cond(R*) rounding."""
    res = rg.synth_gmp(rg.SynthSpec(m=60, p=50, n=20, rank_frac=0.7, seed=2, field="real"))
    spec = rg.compute_gsv(res.pair, rg.GsvOptions(method="direct"))
    tol = 1e-13 * max(res.condition_r, 1.0) * 10
    assert (spec.r, spec.s) == (res.true_spectrum.r, res.true_spectrum.s)
    assert np.max(np.abs(spec.alphas - res.true_spectrum.alphas)) <= tol
    assert np.max(np.abs(spec.betas - res.true_spectrum.betas)) <= tol


def test_run_bench_records():
    cfg = hb.RunConfig(synth=rg.SynthSpec(m=80, p=60, n=24, rank_frac=0.75, seed=4, field="real"),
                       options=rg.GsvOptions(extraction=rg.ExtractionConfig(seed=10)),
                       repetitions=3)
    recs = rg.run_bench(cfg)
    assert [r.method for r in recs] == ["direct"] * 3 + ["randomized"] * 3
    assert [r.repetition for r in recs] == [0, 1, 2, 0, 1, 2]
    for r in recs:
        assert (r.m, r.p, r.n) == (80, 60, 24) and r.seconds > 0.0
    d, z = recs[0], recs[3]
    assert d.err_alpha == 0.0 and d.err_beta == 0.0
    assert d.residual1 is None and d.residual2 is None and (d.l1, d.l2) == (80, 60)
    # the adaptive extraction captures the rank-18 matrices exactly
    assert z.l1 <= 24 and z.l2 <= 24 and z.residual1 is not None
    assert z.err_alpha <= 1e-8 and z.err_beta <= 1e-8
    med = rg.median_seconds(recs)
    assert set(med) == {"direct", "randomized"}
    assert med["direct"] == sorted(r.seconds for r in recs[:3])[1]
    # randomized repetition `rep` uses extraction seed base + rep (bench.py:101-105)
    pair = hb.load_pair(cfg)
    opts = rg.GsvOptions(extraction=rg.ExtractionConfig(seed=12))
    spec2 = rg.compute_gsv(pair, opts)
    truth = rg.compute_gsv(pair, rg.GsvOptions(method="direct"))
    assert abs(float(np.linalg.norm(spec2.alphas - truth.alphas)) - recs[5].err_alpha) <= 1e-13


def test_cli_synth_then_bench(tmp_path, capsys):
    out = tmp_path / "pair"
    rc = cli.main(["synth", "--m", "30", "--p", "24", "--n", "10", "--rank-frac", "0.8",
                   "--seed", "3", "--field", "real", "--out-dir", str(out), "--format", "json"])
    assert rc == 0
    assert "condition_r=" in capsys.readouterr().err
    g1 = rg.read_matrix(out / "g1.mtx")
    assert g1.shape == (30, 10) and (out / "truth.json").exists()
    ref = rg.synth_gmp(rg.SynthSpec(m=30, p=24, n=10, rank_frac=0.8, seed=3, field="real"))
    assert np.array_equal(g1, _host(ref.pair.g1))  # 17 significant digits round-trip
    rep = tmp_path / "bench.csv"
    rc = cli.main(["bench", "--g1", str(out / "g1.mtx"), "--g2", str(out / "g2.mtx"), "--reps",
                   "2", "-o", str(rep)])
    assert rc == 0
    err = capsys.readouterr().err
    assert "median direct:" in err and "median randomized:" in err
    lines = rep.read_text().splitlines()
    assert lines[0].startswith("method,repetition,seconds") and len(lines) == 5
    # the reference's default field is complex: rejected loudly (exit code 5)
    assert cli.main(["synth", "--m", "30", "--p", "24", "--n", "10", "--out-dir", str(out)]) == 5
    assert cli.main(["bench", "--m", "30", "--p", "24"]) == 5


def test_synth_large_pair_spectrum_recovered():
    """A size beyond the Householder route (rows > 1408: CholeskyQR3 left
    blocks, 128-wide GEMM tiles): orthogonality of the construction shows in
    the direct method recovering the prescribed spectrum."""
    res = rg.synth_gmp(rg.SynthSpec(m=3000, p=2500, n=600, rank_frac=0.7, seed=9, field="real"))
    assert res.pair.m == 3000 and res.pair.p == 2500 and res.pair.n == 600
    spec = rg.compute_gsv(res.pair, rg.GsvOptions(method="direct"))
    assert (spec.r, spec.s) == (res.true_spectrum.r, res.true_spectrum.s) == (180, 240)
    tol = 1e-13 * res.condition_r * 10
    assert np.max(np.abs(spec.alphas - res.true_spectrum.alphas)) <= tol
    assert np.max(np.abs(spec.betas - res.true_spectrum.betas)) <= tol
