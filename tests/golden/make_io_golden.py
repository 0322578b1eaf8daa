"""Generate tests/golden/io/ by running the REFERENCE's I/O layer and command
line (rgsv 0.1.0, io.py:30-264, cli.py:88-176) here; the tests only read the
committed files.

    python tests/golden/make_io_golden.py

Inputs: the reference test_cli.py pair (gaussian_matrix(24, 12, seed=1) /
(20, 12, seed=2), test_cli.py:26-32), written with the reference's
write_matrix. Outputs, each produced by the reference's own `main`:
  gsv_direct.csv / .json          gsv --method direct
  gsv_seed9.csv                   gsv --seed 9 (adaptive default options)
  compare_seed7.json / .csv       compare --seed 7
  extract_bs4.json / .csv         extract --input g1 --blocksize 4
  bounds_k4.json / .csv           bounds --k 4 --oversample 3 --tol 1e-12
plus a coordinate / symmetric Matrix Market sample written by scipy
(coord_sym.mtx, with its dense form in coord_sym.npy).
"""

import contextlib
import io as _io
import os
import sys

import numpy as np
import scipy.io
import scipy.sparse

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "io")
sys.path.insert(0, "/root/reference/pkg/src")

import rgsv  # noqa: E402  (the reference)
from rgsv import cli  # noqa: E402

os.makedirs(OUT, exist_ok=True)
g1p, g2p = os.path.join(OUT, "g1.mtx"), os.path.join(OUT, "g2.mtx")
rgsv.write_matrix(g1p, rgsv.gaussian_matrix(24, 12, seed=1))
rgsv.write_matrix(g2p, rgsv.gaussian_matrix(20, 12, seed=2))


def run(name, *argv):
    err = _io.StringIO()
    with contextlib.redirect_stderr(err):
        rc = cli.main([*argv, "-o", os.path.join(OUT, name)])
    assert rc == 0, (name, rc, err.getvalue())
    return err.getvalue()


pair = ["--g1", g1p, "--g2", g2p]
for fmt in ("csv", "json"):
    run(f"gsv_direct.{fmt}", "gsv", *pair, "--method", "direct", "--format", fmt)
    run(f"compare_seed7.{fmt}", "compare", *pair, "--seed", "7", "--format", fmt)
    run(f"extract_bs4.{fmt}", "extract", "--input", g1p, "--blocksize", "4", "--format", fmt)
    err = run(f"bounds_k4.{fmt}", "bounds", *pair, "--k", "4", "--oversample", "3", "--tol",
              "1e-12", "--format", fmt)
run("gsv_seed9.csv", "gsv", *pair, "--seed", "9")
with open(os.path.join(OUT, "bounds_k4.stderr"), "w") as fh:
    fh.write(err)

rng = np.random.default_rng(5)
low = np.tril(rng.standard_normal((6, 6)))
low[np.abs(low) < 0.6] = 0.0
scipy.io.mmwrite(os.path.join(OUT, "coord_sym.mtx"), scipy.sparse.coo_matrix(low),
                 symmetry="symmetric", precision=17)
np.save(os.path.join(OUT, "coord_sym.npy"), low + np.tril(low, -1).T)
print(sorted(os.listdir(OUT)))
