"""Generate tests/golden/*.npz from the REAL reference package.

Run in the build container only (needs /root/reference):

    python tests/golden/make_golden.py

It builds the reference package in a scratch copy (/tmp/refbuild, the recipe
of SURVEY.md 8c), imports it, and records outputs of its own public API
(`pcd_fit`, `cd_fit`, `compute_gram`, `build_circle_schedule`, the compiled
`pcd_sweep`) on seeded inputs.  The fixtures are small so they can be
committed; tests/test_oracle.py pins oracle/ against them and the GPU parity
tests compare the CUDA path with them.  Also asserts that
paper_2106_09382_b200.synth reproduces the reference generators bitwise.
"""

import hashlib
import os
import shutil
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
SCRATCH = "/tmp/refbuild"


def _import_reference():
    staged = os.path.join(REPO, "baseline", "_ref", "pkg", "src")  # tools/stage_reference_suite.py (travels)
    if not os.path.isdir("/root/reference") and os.path.isdir(staged):
        sys.path.insert(0, staged)
        import parconcord as pc

        assert pc.HAVE_COMPILED, "staged reference has no compiled backend"
        return pc
    pkg = os.path.join(SCRATCH, "pkg")
    if not os.path.isdir(pkg):
        os.makedirs(SCRATCH, exist_ok=True)
        shutil.copytree("/root/reference/pkg", pkg)
        subprocess.run(["chmod", "-R", "u+w", pkg], check=True)
        env = dict(os.environ, CC="/usr/bin/gcc", LDSHARED="/usr/bin/gcc -shared")
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"],
                       cwd=pkg, env=env, check=True, capture_output=True)
    sys.path.insert(0, os.path.join(pkg, "src"))
    import parconcord as pc

    assert pc.HAVE_COMPILED, "reference compiled backend did not build"
    return pc


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    pc = _import_reference()
    sys.path.insert(0, REPO)
    from paper_2106_09382_b200 import synth

    out = {}

    # --- schedule known answers (test_schedule.py:18-27, test_acceptance.py:73-91)
    for p in list(range(2, 21)) + [101]:
        sched = pc.build_circle_schedule(p)
        from parconcord.solver import _flatten_schedule

        rs, ss, off = _flatten_schedule(sched)
        out[f"sched_{p}_rs"] = rs.astype(np.int64)
        out[f"sched_{p}_ss"] = ss.astype(np.int64)
        out[f"sched_{p}_off"] = off.astype(np.int64)

    # --- Gram / soft threshold known answers (test_model.py:50-54, 107-116)
    g = pc.compute_gram(pc.DataMatrix(np.array([[1.0, 2.0], [3.0, 4.0]])))
    out["gram_2x2"] = g.t
    xs = np.array([3.0, -3.0, 0.5, -0.5, 1.0, -1.0, 0.0, 2.5])
    out["soft_x"] = xs
    out["soft_tau1"] = np.array([pc.soft_threshold(float(v), 1.0) for v in xs])

    # --- full fits through the reference's public API, compiled backend
    cases = [
        ("ar2_p100_n50_l0.3", "ar2", 100, 50, 0.3, 1e-5, True),
        ("ar2_p100_n50_l0.1", "ar2", 100, 50, 0.1, 1e-5, False),
        ("ar2_p100_n50_l0.3_tol1e-8", "ar2", 100, 50, 0.3, 1e-8, False),
        ("sf_p101_n50_l0.3", "scale_free", 101, 50, 0.3, 1e-5, True),
        ("ar2_p9_n70_l0.1", "ar2", 9, 70, 0.1, 1e-6, True),
        ("ar2_p12_n60_l0.1_tol1e-8", "ar2", 12, 60, 0.1, 1e-8, False),
    ]
    names = []
    for name, kind, p, n, lam, tol, keep_sweeps in cases:
        truth = pc.ar2_precision(p) if kind == "ar2" else pc.scale_free_precision(p, seed=0)
        raw = pc.sample_mvn(truth, n, seed=0)
        data = pc.center_columns(raw)
        gram = pc.compute_gram(data)
        # our host generators must reproduce the reference bitwise
        mine_truth = synth.ar2_precision(p) if kind == "ar2" else synth.scale_free_precision(p, seed=0)
        assert np.array_equal(mine_truth, truth.omega_true.omega), name
        assert np.array_equal(synth.sample_mvn(mine_truth, n, seed=0), raw.values), name
        assert np.array_equal(synth.center(raw.values), data.values), name
        assert np.array_equal(synth.host_gram(data.values), gram.t), name

        cfg = pc.SolverConfig(lam=lam, delta_tol=tol, max_outer_iterations=5000)
        rep = pc.pcd_fit(gram, cfg, backend="compiled")
        cd = pc.cd_fit(gram, cfg, backend="compiled")
        out[f"{name}_x"] = data.values
        out[f"{name}_t"] = gram.t
        out[f"{name}_meta"] = np.array([p, n, lam, tol])
        out[f"{name}_omega"] = rep.estimate.omega
        out[f"{name}_iters"] = np.array(rep.iterations)
        out[f"{name}_delta"] = np.array(rep.final_delta)
        out[f"{name}_edges"] = np.array(rep.edge_count)
        out[f"{name}_obj"] = np.array(rep.objective_trace)
        out[f"{name}_cd_omega"] = cd.estimate.omega
        out[f"{name}_cd_iters"] = np.array(cd.iterations)
        if keep_sweeps:
            be = pc.get_backend("compiled")
            from parconcord.solver import _flatten_schedule

            rs, ss, off = _flatten_schedule(pc.build_circle_schedule(p))
            om = np.eye(p)
            for k in range(3):
                be.pcd_sweep(om, gram.t, float(gram.n), gram.n * lam, rs, ss, off, 1)
                out[f"{name}_sweep{k + 1}"] = om.copy()
        names.append(name)
        print(f"{name}: iters={rep.iterations} edges={rep.edge_count} "
              f"delta={rep.final_delta:.3e} cd_iters={cd.iterations}")

    # --- larger configs (configs[1]): summaries only.  T is the portable exact Gram
    # (synth.portable_problem: X rounded onto a grid where X^T X is exact in FP64), so the GPU
    # box regenerates the same bits from the seed; the reference's compute_gram gives that T too.
    summaries = []
    for row, (kind, p, n, lam) in enumerate([("scale_free", 1000, 500, 0.3), ("scale_free", 1001, 500, 0.3),
                                             ("ar2", 1000, 500, 0.3), ("scale_free", 1000, 500, 0.1),
                                             ("scale_free", 1001, 500, 0.1), ("ar2", 1001, 500, 0.1)]):
        x, t = synth.portable_problem(kind, p, n, seed=0)
        assert np.array_equal(pc.compute_gram(pc.DataMatrix(x)).t, t)
        gram = pc.GramMatrix(t, n)
        cfg = pc.SolverConfig(lam=lam, delta_tol=1e-5, max_outer_iterations=5000, workers=8)
        rep = pc.pcd_fit(gram, cfg, backend="compiled")
        summaries.append([0 if kind == "ar2" else 1, p, n, lam, rep.iterations, rep.edge_count,
                          rep.final_delta, rep.objective_trace[-1]])
        out[f"big_{row}_tsha"] = np.frombuffer(sha(gram.t).encode(), np.uint8)
        out[f"big_{row}_omsha"] = np.frombuffer(sha(rep.estimate.omega).encode(), np.uint8)
        print(f"big {kind} p={p} lam={lam}: iters={rep.iterations} edges={rep.edge_count}")
    out["big_summary"] = np.array(summaries)
    out["case_names"] = np.array(names)

    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)
    print("wrote", os.path.join(HERE, "reference_golden.npz"))


if __name__ == "__main__":
    main()
