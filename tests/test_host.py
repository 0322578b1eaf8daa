"""Host-side logic of the drop-in API (no device needed)."""

import math

import numpy as np
import pytest

from paper_2404_09459_b200 import (
    ExtractionConfig,
    GsvOptions,
    GsvSpectrum,
    ValidationError,
    DimensionError,
    classify_spectrum,
    gaussian_matrix,
)
from paper_2404_09459_b200.rangefinder import single_block_width
from paper_2404_09459_b200.workloads import CONFIGS, make_pair


def test_config_validation_mirrors_reference():
    with pytest.raises(ValidationError):
        ExtractionConfig(tol=0.0)
    with pytest.raises(ValidationError):
        ExtractionConfig(blocksize=0)
    with pytest.raises(ValidationError):
        ExtractionConfig(trim_tol=-1e-3)
    with pytest.raises(ValidationError):
        ExtractionConfig(max_cols=0)
    with pytest.raises(ValidationError):
        ExtractionConfig(power_iters=-1)
    with pytest.raises(ValidationError):
        GsvOptions(classify_tol=0.5)
    with pytest.raises(ValidationError):
        GsvOptions(method="magic")
    # fp32 compute mode (not in the reference, which promotes to fp64)
    assert GsvOptions().f32_mode == "tf32x3"
    assert GsvOptions(f32_mode="promote").f32_mode == "promote"
    with pytest.raises(ValidationError):
        GsvOptions(f32_mode="fp16")


def test_single_block_detection():
    fixed = ExtractionConfig.fixed_rank(30, seed=0, power_iters=1)
    assert single_block_width(fixed, 2000, 200) == 30
    assert single_block_width(ExtractionConfig(blocksize=500, trim_tol=0.0), 50, 200) == 200
    # adaptive default (trim on, several blocks) is not a single block
    assert single_block_width(ExtractionConfig(), 2000, 200) is None
    assert single_block_width(ExtractionConfig(blocksize=10, max_cols=30, trim_tol=0.0),
                              100, 50) is None


def test_spectrum_invariants():
    with pytest.raises(ValidationError):
        GsvSpectrum(np.array([0.9, 0.5]), np.array([0.9, 0.5]), r=0, s=2)
    with pytest.raises(ValidationError):
        GsvSpectrum(np.array([0.5, 0.9]), np.sqrt(1 - np.array([0.5, 0.9]) ** 2), r=0, s=2)
    with pytest.raises(ValidationError):
        GsvSpectrum(np.array([1.0, 0.5]), np.array([1e-13, math.sqrt(0.75)]), r=1, s=1)
    with pytest.raises(DimensionError):
        GsvSpectrum(np.array([]), np.array([]), r=0, s=0)
    spec = GsvSpectrum(np.array([1.0, 0.6, 0.0]), np.array([0.0, 0.8, 1.0]), 1, 1)
    assert spec.n == 3


def test_classify_snaps_in_place():
    a = np.array([1.0 - 1e-13, 0.6, 1e-12])
    b = np.array([5e-13, 0.8, 1.0 - 1e-14])
    assert classify_spectrum(a, b, 1e-10) == (1, 1)
    assert a[0] == 1.0 and b[0] == 0.0 and a[2] == 0.0 and b[2] == 1.0
    with pytest.raises(ValidationError):
        classify_spectrum(np.array([1.0]), np.array([0.0]), classify_tol=0.5)


def test_gaussian_matrix_reference_convention():
    g = gaussian_matrix(5, 3, 7)
    assert np.array_equal(g, np.random.default_rng(7).standard_normal((5, 3)))
    c = gaussian_matrix(4, 2, 1, "complex")
    assert np.iscomplexobj(c)
    with pytest.raises(ValidationError):
        gaussian_matrix(2, 2, 0, "quaternion")
    with pytest.raises(DimensionError):
        gaussian_matrix(0, 2, 0)


def test_workload_generator():
    cfg = CONFIGS["cfg0"]
    g1, g2 = make_pair(cfg)
    assert g1.shape == (2000, 200) and g2.shape == (1500, 200)
    h1, _ = make_pair(cfg)
    assert np.array_equal(g1, h1)
    s = np.linalg.svd(g1, compute_uv=False)
    assert s[19] > 1e3 * s[20]  # rank-20 signal over 1e-8 noise
    assert CONFIGS["cfg1"].flops == 2.0 * 36000 * 1000 * 60 * 6
    assert CONFIGS["cfg3"].batch == 4096


# ------------------------------------------------ routing and batch results
def test_mode_routing():
    """fixed-width -> fused pair pipeline; direct / adaptive -> general loop."""
    from paper_2404_09459_b200.engine import _fixed_width

    fixed = GsvOptions(extraction=ExtractionConfig.fixed_rank(30, 0, 1))
    assert _fixed_width(fixed, 2000, 1500, 200) == (30, 30)
    assert _fixed_width(GsvOptions(), 2000, 1500, 200) is None          # adaptive default
    assert _fixed_width(GsvOptions(method="direct"), 20, 15, 30) is None  # no extraction
    # direct ignores max_cols like the reference (engine.py:246-249)
    big = GsvOptions(method="direct", extraction=ExtractionConfig(max_cols=500))
    assert _fixed_width(big, 20, 15, 30) is None
    with pytest.raises(ValidationError):
        _fixed_width(GsvOptions(extraction=ExtractionConfig(max_cols=500)), 20, 15, 30)


class _FakePlan:
    def __init__(self, B, n, k):
        self.B, self.n, self.k = B, n, k
        self.res_stride = 6 * n + 4 + 2 * k


def _fake_batch(B=3, n=8, k=2):
    """Host buffers laid out like rgsv_batch_gsvd's outputs (F2 spectra)."""
    plan = _FakePlan(B, n, k)
    rs = plan.res_stride
    fh = np.zeros(B * rs + 4 * B)
    ih = np.zeros(5 * B, dtype=np.int32)
    for j in range(B):
        o = fh[j * rs:(j + 1) * rs]
        o[:k] = 1.0                      # alphas
        o[n + k:2 * n] = 1.0             # betas
        o[2 * n:2 * n + k] = np.inf      # rho
        o[4 * n:4 * n + k] = 1.0 / k     # p1
        o[5 * n + k:6 * n] = 1.0 / (n - k)
        o[6 * n:6 * n + 4] = [math.log(k) / math.log(n), math.log(n - k) / math.log(n), 1, 1]
        o[6 * n + 4:6 * n + 4 + 2 * k] = 1.0
        ih[4 * j:4 * j + 4] = [k, k, k, 0]
        fh[B * rs + 4 * j:B * rs + 4 * j + 4] = [10.0 + j, 4.0, 9.0, 2.0]
    return fh, ih, plan


def test_small_batch_runs_vectorized_validation():
    from paper_2404_09459_b200.engine import SmallBatchRuns

    fh, ih, plan = _fake_batch()
    runs = SmallBatchRuns(fh, ih, plan, GsvOptions(extraction=ExtractionConfig.fixed_rank(2)))
    assert len(runs) == 3
    r1 = runs[1]
    assert (r1.r, r1.s) == (2, 0) and np.array_equal(r1.alphas, [1, 1, 0, 0, 0, 0, 0, 0])
    assert r1.basis1.residual_history == [math.sqrt(11.0), math.sqrt(7.0)]
    assert r1.d1 == pytest.approx(math.log(2) / math.log(8))
    assert [r.r for r in runs[0:3]] == [2, 2, 2] and runs[-1].r == 2
    with pytest.raises(IndexError):
        runs[3]


@pytest.mark.parametrize("corrupt,exc", [
    ("pythagoras", ValidationError),
    ("order", ValidationError),
    ("unsnapped", ValidationError),
    ("chol", "RankDeficiencyError"),
    ("jacobi", "ConvergenceError"),
    ("nonfinite", ValidationError),
])
def test_small_batch_runs_reject(corrupt, exc):
    import paper_2404_09459_b200 as rg
    from paper_2404_09459_b200.engine import SmallBatchRuns

    fh, ih, plan = _fake_batch()
    n, rs = plan.n, plan.res_stride
    o = fh[rs:2 * rs]
    if corrupt == "pythagoras":
        o[n + 3] = 0.5
    elif corrupt == "order":
        o[1], o[2] = 0.5, 0.9
        o[n + 1], o[n + 2] = math.sqrt(0.75), math.sqrt(1 - 0.81)
    elif corrupt == "unsnapped":
        o[n + 0] = 1e-300  # classified-zero beta that is not exactly 0
        o[0] = math.sqrt(1 - 1e-600)
    elif corrupt == "chol":
        ih[4 * 3 + 1] = 0x1
    elif corrupt == "jacobi":
        ih[4 * 3 + 2] = 0x4
    elif corrupt == "nonfinite":
        fh[3 * rs + 4] = np.nan
    if corrupt in ("pythagoras", "order", "unsnapped"):
        ih[4 * 3 + 1] = 0x80  # RGSV_ST_SPECTRUM: k_batch_small's device-side check
    exc = getattr(rg, exc) if isinstance(exc, str) else exc
    with pytest.raises(exc):
        SmallBatchRuns(fh, ih, plan, GsvOptions(extraction=ExtractionConfig.fixed_rank(2)))


def test_small_batch_runs_spectrum_message_and_nan():
    """The host re-scan behind RGSV_ST_SPECTRUM names the violated invariant
    with the reference's message; a NaN spectrum (no numpy comparison
    catches it) still raises."""
    from paper_2404_09459_b200.engine import SmallBatchRuns

    opts = GsvOptions(extraction=ExtractionConfig.fixed_rank(2))
    fh, ih, plan = _fake_batch()
    n, rs = plan.n, plan.res_stride
    fh[rs + n] = 1e-300  # classified-zero beta that is not exactly 0
    fh[rs] = math.sqrt(1 - 1e-600)
    ih[4 * 3 + 1] = 0x80
    with pytest.raises(ValidationError, match="classified-zero"):
        SmallBatchRuns(fh, ih, plan, opts)
    fh, ih, plan = _fake_batch()
    fh[2 * rs] = np.nan  # alpha_0 of pair 2
    ih[4 * 3 + 2] = 0x80
    with pytest.raises(ValidationError, match="GSVs must lie"):
        SmallBatchRuns(fh, ih, plan, opts)


def test_bench_reference_arm_contract():
    """bench.py --impl reference prints one JSON line with the contract keys
    (the oracle port timed on the host cores)."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference",
                          "--config", "cfg0", "--steps", "2", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e", "impl"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"


def test_sharded_bench_mode_is_wired():
    """bench.py's default is cfg2; N > 1 routes single-pair configs to the
    row-sharded strong-scaling driver (dist.compute_gsv_sharded)."""
    import os
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import bench
    from paper_2404_09459_b200 import dist as rdist

    sys.argv = ["bench.py", "--sharded", "--config", "cfg4"]
    args = bench.parse()
    assert args.sharded and args.config == "cfg4"
    assert bench.select_mode(args, 1) == "sharded"
    sys.argv = ["bench.py"]
    args = bench.parse()
    assert args.config == "cfg2"  # the metric's config by default
    assert bench.select_mode(args, 1) == "pairs"
    assert bench.select_mode(args, 8) == "sharded"  # strong scaling at N > 1
    sys.argv = ["bench.py", "--replicas"]
    assert bench.select_mode(bench.parse(), 8) == "pairs"
    sys.argv = ["bench.py", "--config", "cfg3"]
    assert bench.select_mode(bench.parse(), 8) == "batch"
    assert callable(bench.run_ours_sharded) and callable(rdist.compute_gsv_sharded)
    # balanced contiguous gene blocks of the genome-scale configs
    for cfg in ("cfg2", "cfg4"):
        m = CONFIGS[cfg].m
        blocks = [rdist.shard_rows(m, r, 8) for r in range(8)]
        assert blocks[0][0] == 0 and blocks[-1][1] == m


def test_projector_bound_host_formula_matches_reference_golden():
    """projector_bound is O(n) host math on top of the device-validated
    stacked norm: with the reference's own stack_norm2 and spectrum it
    reproduces the reference's certificates (tests/golden/ref_bounds.npz)."""
    import os
    from types import SimpleNamespace

    from paper_2404_09459_b200.bounds import projector_bound

    gold = np.load(os.path.join(os.path.dirname(__file__), "golden", "ref_bounds.npz"))
    for c in (0, 1):
        g1, g2 = gold[f"c{c}_g1"], gold[f"c{c}_g2"]
        pair = SimpleNamespace(m=g1.shape[0], p=g2.shape[0], n=g1.shape[1],
                               stack_norm2=float(gold[f"c{c}_stack_norm2"]))
        spec = SimpleNamespace(alphas=gold[f"c{c}_alphas"], betas=gold[f"c{c}_betas"])
        for k, os_, side, want in gold[f"c{c}_projector"]:
            got = projector_bound(pair, spec, k=int(k), oversample=int(os_),
                                  which="first" if side == 0 else "second")
            assert got == want or abs(got - want) <= 1e-14 * abs(want)


def test_synth_spec_and_run_config_validation():
    """SynthSpec / RunConfig argument checks and messages of the reference
    (synthetic.py:36-49, bench.py:31-42); no device needed."""
    import paper_2404_09459_b200 as rg

    spec = rg.SynthSpec(m=10, p=8, n=6)
    assert spec.rank == 3 and spec.field == "complex" and spec.rank_frac == 0.6
    for kw, msg in ((dict(m=0, p=1, n=2), "m and p must be >= 1"), (dict(m=1, p=1, n=1), "n must be"),
                    (dict(m=2, p=2, n=2, rank_frac=0.0), "rank_frac"),
                    (dict(m=2, p=2, n=2, rank_frac=1.5), "rank_frac"),
                    (dict(m=2, p=2, n=2, field="quaternion"), "field must be")):
        with pytest.raises(rg.ValidationError, match=msg):
            rg.SynthSpec(**kw)
    with pytest.raises(rg.InfeasibleRankError):
        rg.synth_gmp(rg.SynthSpec(m=10, p=8, n=6, rank_frac=0.3, field="real"))
    with pytest.raises(rg.ValidationError, match="yields empty"):
        rg.synth_gmp(rg.SynthSpec(m=1, p=1, n=4, rank_frac=0.5, field="real"))
    with pytest.raises(rg.ValidationError, match="complex"):
        rg.synth_gmp(spec)

    with pytest.raises(rg.ValidationError, match="given together"):
        rg.RunConfig(g1_path="a.mtx")
    with pytest.raises(rg.ValidationError, match="exactly one input source"):
        rg.RunConfig()
    with pytest.raises(rg.ValidationError, match="exactly one input source"):
        rg.RunConfig(g1_path="a", g2_path="b", synth=spec)
    with pytest.raises(rg.ValidationError, match="repetitions"):
        rg.RunConfig(synth=spec, repetitions=0)
    with pytest.raises(rg.ValidationError, match="format"):
        rg.RunConfig(synth=spec, format="xml")
    cfg = rg.RunConfig(synth=spec)
    assert cfg.options == rg.GsvOptions() and cfg.repetitions == 1 and cfg.format == "csv"

    recs = [rg.BenchRecord("direct", i, s, 0.0, 0.0, None, None, 4, 4, 4, 4, 2)
            for i, s in enumerate((3.0, 1.0, 2.0))]
    recs.append(rg.BenchRecord("randomized", 0, 5.0, 0.0, 0.0, 1e-9, 1e-9, 2, 2, 4, 4, 2))
    assert rg.median_seconds(recs) == {"direct": 2.0, "randomized": 5.0}


def test_true_spectrum_layout():
    """alpha = (ones, interior, zeros), beta exact 0 / 1 in the outer blocks
    (synthetic.py:85-89)."""
    from paper_2404_09459_b200.synthetic import true_spectrum

    sp = true_spectrum(6, 4, np.array([0.8, 0.3]))
    assert (sp.r, sp.s, sp.n) == (2, 2, 6)
    assert list(sp.alphas) == [1.0, 1.0, 0.8, 0.3, 0.0, 0.0]
    assert list(sp.betas[:2]) == [0.0, 0.0] and list(sp.betas[4:]) == [1.0, 1.0]
    assert np.allclose(sp.alphas**2 + sp.betas**2, 1.0, atol=1e-15)
