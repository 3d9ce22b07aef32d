"""Golden vectors for the boundary formats and diagnostics, from the REAL reference.

Run in the build container only (needs /root/reference, reuses make_golden's build):

    python tests/golden/make_golden_io.py

Records, on the estimates of reference_golden.npz:
  * the text the reference's fileio.write_estimate / write_problem produce;
  * the reference's check_optimality report (worst violation, coordinate).
"""

import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import _import_reference  # noqa: E402


def main():
    pc = _import_reference()
    from parconcord import fileio

    g = np.load(os.path.join(HERE, "reference_golden.npz"))
    out = {}
    with tempfile.TemporaryDirectory() as td:
        for name in [str(s) for s in g["case_names"]]:
            p, n, lam, tol = g[f"{name}_meta"]
            est = pc.PrecisionEstimate(g[f"{name}_omega"])
            gram = pc.GramMatrix(g[f"{name}_t"], int(n))
            rep = pc.check_optimality(est, gram, float(lam))
            out[f"{name}_opt"] = np.array([rep.worst_violation, rep.worst_coordinate[0], rep.worst_coordinate[1]])
            path = os.path.join(td, "e.txt")
            fileio.write_estimate(path, est, float(lam), int(g[f"{name}_iters"]), float(g[f"{name}_delta"]))
            out[f"{name}_estimate_txt"] = np.frombuffer(open(path, "rb").read(), np.uint8)
        path = os.path.join(td, "x.txt")
        fileio.write_problem(path, pc.DataMatrix(g["ar2_p9_n70_l0.1_x"], centered=True))
        out["ar2_p9_n70_l0.1_problem_txt"] = np.frombuffer(open(path, "rb").read(), np.uint8)
    np.savez_compressed(os.path.join(HERE, "reference_io_golden.npz"), **out)
    print("wrote", os.path.join(HERE, "reference_io_golden.npz"), sorted(out)[:4], "...")


if __name__ == "__main__":
    main()
