"""Cold-path (tridiagonal) PSD projection checks on the GPU.

    python tools/cold_check.py [--iters 40]

A: project_cone on random and adversarial symmetric blocks (d = 33 .. 111)
   against numpy's eigh projection.
B: config 4, per-iteration time and split statistics of the first iterations,
   cold path vs the Jacobi variant (HSDE_FLAG_JACOBI), and the iterate gap.
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_1611_01828_b200 as H  # noqa: E402
from paper_1611_01828_b200 import _lib  # noqa: E402
from paper_1611_01828_b200.problem import CliqueDecomposition, DecomposedProblem  # noqa: E402
from paper_1611_01828_b200.synthetic import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=40)
ap.add_argument("--skip-b", action="store_true")
a = ap.parse_args()


def proj(b):
    w, v = np.linalg.eigh(0.5 * (b + b.T))
    return (v * np.maximum(w, 0.0)) @ v.T


def blocks(rng, d):
    q, _ = np.linalg.qr(rng.normal(size=(d, d)))
    out = {"random": rng.normal(size=(d, d))}
    lam = np.ones(d); lam[: d // 3] = -2.0
    out["two_values"] = (q * lam) @ q.T
    lam = np.linspace(-1, 1, d); lam[d // 2: d // 2 + 5] = 1e-13 * np.arange(5)
    out["near_zero_cluster"] = (q * lam) @ q.T
    out["identity"] = np.eye(d)
    out["diag"] = np.diag(rng.normal(size=d))
    out["zero"] = np.zeros((d, d))
    x = rng.normal(size=d)
    out["rank1"] = np.outer(x, x) - 0.5 * np.eye(d)
    lam = np.concatenate([1 + 1e-9 * rng.normal(size=d // 2), -1 + 1e-9 * rng.normal(size=d - d // 2)])
    out["tight_clusters"] = (q * lam) @ q.T
    out["graded"] = (q * np.logspace(-12, 0, d) * np.sign(rng.normal(size=d))) @ q.T
    return out


rng = np.random.default_rng(7)
sizes = [33, 40, 47, 64, 80, 81, 84, 85, 96, 111]
kinds = list(blocks(rng, 40).keys())
worst = 0.0
for kind in kinds:
    n = sum(sizes)
    cl, o = [], 0
    for d in sizes:
        cl.append(list(range(o, o + d)))
        o += d
    dec = CliqueDecomposition.build(n, cl)
    A = sp.csr_matrix(([1.0], ([0], [0])), shape=(1, n * n))
    dp = DecomposedProblem(n=n, m=1, c=np.eye(n).ravel(), A=A, b=np.ones(1), dec=dec, block_dims=(n,))
    _, layout = H.build_hsde(dp)
    u = rng.normal(size=layout.total)
    s = u[layout.sl_s]
    for k, d in enumerate(sizes):
        s[dec.offsets[k]:dec.offsets[k + 1]] = blocks(rng, d)[kind].ravel()
    u[layout.sl_s] = s
    got = H.project_cone(u, layout)[layout.sl_s]
    errs = []
    for k, d in enumerate(sizes):
        o0, o1 = dec.offsets[k], dec.offsets[k + 1]
        want = proj(s[o0:o1].reshape(d, d)).ravel()
        e = np.linalg.norm(got[o0:o1] - want) / max(np.linalg.norm(s[o0:o1]), 1e-300)
        errs.append(e)
        worst = max(worst, e)
    print(f"A {kind:18s}", " ".join(f"{d}:{e:.1e}" for d, e in zip(sizes, errs)), flush=True)
print("A worst rel err", worst, flush=True)

if not a.skip_b:
    cp = make_config(4)
    res = {}
    for name, flags in (("cold", 0), ("jacobi", _lib.HSDE_FLAG_JACOBI)):
        h = _lib.Handle(cp, flags=flags)
        t0 = time.time()
        line = []
        for i in range(a.iters):
            ms = h.time_iterations(1)
            st = h.stats()
            line.append(f"{i + 1}:{ms:.3f}/{st['split_done']:.2f}/{st['cold_done']:.2f}/{st['cold_failed']:.2f}")
        print(name, "ms/split/cold/fail per iteration:", " ".join(line), flush=True)
        ms = h.time_iterations(20) / 20
        prof, nl = h.profile_iterations(5)
        print(name, f"steady ms/it {ms:.4f}", {k: round(v / 5, 4) for k, v in prof.items() if v}, flush=True)
        res[name] = h.get_state()
        h.close()
    du = np.linalg.norm(res["cold"][0] - res["jacobi"][0]) / np.linalg.norm(res["jacobi"][0])
    print(f"B iterate gap cold vs jacobi after {a.iters + 25} iterations: {du:.3e}")
