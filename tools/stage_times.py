"""Stage timing of one cfg pair: each chain alone, both chains concurrently
(two streams), and the post-join small-GSVD + comparative stage."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2404_09459_b200 as rg  # noqa: E402
from paper_2404_09459_b200 import device as dv  # noqa: E402
from paper_2404_09459_b200 import _native  # noqa: E402
from paper_2404_09459_b200.workloads import CONFIGS, make_pair  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg1"]
g1, g2 = make_pair(cfg)
pair = rg.GmpPair.resident(torch.from_numpy(g1).cuda(), torch.from_numpy(g2).cuda())
plan = dv.pair_plan(cfg.m, cfg.p, cfg.n, cfg.k, cfg.k)
pk = plan.pk
main = torch.cuda.current_stream()
L = _native.lib()


def timed(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def chain1():
    plan.s1.enqueue_omega(pk.d("status"), main)
    plan.s1.launch(pair.g1, cfg.q, pk.d("stats1"), pk.d("rdiag1"), pk.d("status"), main)


def chain2():
    plan.s2.enqueue_omega(pk.d("status"), main)
    plan.s2.launch(pair.g2, cfg.q, pk.d("stats2"), pk.d("rdiag2"), pk.d("status"), main)


def both():
    plan.side.wait_stream(main)
    plan.s1.enqueue_omega(pk.d("status"), main)
    plan.s2.enqueue_omega(pk.d("status"), plan.side)
    plan.s1.launch(pair.g1, cfg.q, pk.d("stats1"), pk.d("rdiag1"), pk.d("status"), main)
    plan.s2.launch(pair.g2, cfg.q, pk.d("stats2"), pk.d("rdiag2"), pk.d("status"), plan.side)
    main.wait_stream(plan.side)


def small():
    L.rgsv_small_gsvd(dv.vp(plan.s1.b), plan.s1.ldb, plan.k1, dv.vp(plan.s2.b), plan.s2.ldb,
                      plan.k2, plan.n, dv.vp(pk.d("sv1")), dv.vp(pk.d("sv2")),
                      dv.vp(pk.d("nsv")), dv.vp(pk.d("status")), dv.vp(plan.small_ws),
                      plan.small_bytes, dv.sp(main))
    L.rgsv_comparative(dv.vp(pk.d("sv1")), dv.vp(pk.d("nsv")), dv.vp(pk.d("sv2")), plan.n, 1e-10,
                       dv.vp(pk.d("alphas")), dv.vp(pk.d("betas")), dv.vp(pk.d("rho")),
                       dv.vp(pk.d("theta")), dv.vp(pk.d("p1")), dv.vp(pk.d("p2")),
                       dv.vp(pk.d("scalars")), dv.vp(pk.d("counts")), dv.vp(pk.d("status")),
                       dv.sp(main))


opts = rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(cfg.k, 0, cfg.q))
full = timed(lambda: plan.run(pair.g1, pair.g2, 0, cfg.q, 1e-10))
print(f"{cfg.name}: chain1 {timed(chain1):8.1f} us | chain2 {timed(chain2):8.1f} us | "
      f"both (2 streams) {timed(both):8.1f} us | small+comparative {timed(small):8.1f} us | "
      f"full graph step {full:8.1f} us")
