"""Write tests/golden/oracle_<CFG>[_tolX][_firstK].json from the ORACLE only (no CUDA path involved).

    python tests/golden/make_oracle_golden.py C3 [C4 ...] [--cycles K] [--tol TOL] [--verbose]

Stores the oracle's eigenvalues, residuals, status, counters and per-cycle log
(t, cumulative A-matvecs, theta_t, ||r_t||, basis width, X^prev width) of the
full-size BASELINE configs whose oracle solve takes minutes to hours, so the GPU parity
tests can compare trajectories without re-running the oracle, plus the eigenvectors'
entries at the seeded rows inputs.sample_rows(n) (the full vectors are 0.3-8.6 GB).
--cycles K stores a bounded prefix (max_cycles=K) instead of the full solve; --tol runs at a
tighter residual tolerance (the eigenvector-parity runs of SURVEY 8(c.5) step 3).
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1711_10128_b200 import inputs  # noqa: E402


def _opt(argv, flag, conv):
    if flag in argv:
        i = argv.index(flag)
        v = conv(argv[i + 1])
        del argv[i:i + 2]
        return v
    return None


def main(argv):
    argv = list(argv)
    cycles = _opt(argv, "--cycles", int)
    tol = _opt(argv, "--tol", float)
    verbose = "--verbose" in argv
    argv = [a for a in argv if a != "--verbose"]
    for name in argv:
        P = inputs.make(name)
        if tol is not None:
            P.tol = tol
        rows = inputs.sample_rows(P.A.n)
        t0 = time.perf_counter()
        exact = name == "C3"  # d = 0 Laplacian: compare the full vectors with the exact eigenspaces
        r = oracle.solve(P.A, P.B, P.p, P.q, P.l, P.tol, P.sigma, want_vectors=exact,
                         max_cycles=cycles or 5000, sample_rows=rows, verbose=verbose)
        dt = time.perf_counter() - t0
        extra = {}
        if exact:
            sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
            from closed_form import laplace3d_lowest, sin_angle
            lam, V, groups = laplace3d_lowest(P.grid["N"], P.p)
            X = r["eigenvectors"]
            extra = {"exact_groups": groups,
                     "exact_sin_angle": [sin_angle(X[:, g], V[:, g]) for g in groups],
                     "exact_eigenvalues": list(map(float, lam))}
        out = {
            "config": name, "desc": P.desc, "p": P.p, "q": P.q, "l": P.l, "tol": P.tol,
            "source": "oracle/ (orc_trplk_solve) via tests/golden/make_oracle_golden.py",
            "prefix_cycles": cycles,
            "status": r["status"], "cycles": r["cycles"], "a_matvecs": r["a_matvecs"],
            "b_matvecs": r["b_matvecs"], "eigenvalues": list(map(float, r["eigenvalues"])),
            "residuals": list(map(float, r["residuals"])),
            "log": {k: [float(x) if k in ("theta_t", "res") else int(x) for x in v]
                    for k, v in r["log"].items() if k in ("t", "mv", "theta_t", "res", "k", "nprev")},
            "log_thetas": [list(map(float, row)) for row in r["log"]["thetas"]],
            "sample_rows": [int(x) for x in rows],
            "sample_vectors": [list(map(float, r["samples"][:, c])) for c in range(P.p)],
            **extra,
            "oracle_seconds": dt, "host_cores": os.cpu_count(),
            "omp_threads": int(os.environ.get("OMP_NUM_THREADS", os.cpu_count())),
        }
        suffix = (f"_tol{tol:.0e}" if tol is not None else "") + (f"_first{cycles}" if cycles else "")
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"oracle_{name}{suffix}.json")
        json.dump(out, open(path, "w"))
        print(name, r["status"], r["cycles"], r["a_matvecs"], f"{dt:.1f}s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
