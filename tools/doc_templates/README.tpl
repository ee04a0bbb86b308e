# chordal-hsde-b200

This repository holds a from-scratch, B200-native (sm_100a, fp64) implementation of one path: the per-iteration hot path of the homogeneous self-dual embedding (HSDE) ADMM for chordally sparse SDPs from arXiv:1611.01828 (Zheng, Fantuzzi, Papachristodoulou, Goulart, Wynn). It does not re-implement the whole reference package (`chordalsdp`). It keeps that package's `solve_decomposed`/`SolverSettings`/`SolverReport` contract, so the same decomposed `(A, b, C, clique pattern)` goes in, and the same iterates `x, s, y, v, τ/κ`, status, certificate and per-check iteration log come out. Python host code calls hand-written CUDA kernels through a thin C-ABI. Those kernels are:

- vectorised clique gather/scatter (`H x`, `Hᵀ s`);
- batched PSD-cone projections: warp-level Jacobi for cliques up to 32 (`k_cone_warp`); for larger ones a cold path (`k_cone_cold`: Householder tridiagonalisation in registers, bisection, twisted factorisations, compact-WY back transformation and the reconstruction on fp64 `mma.sync` DMMA) and a warm path (`k_cone_split`: projection onto a kept invariant subspace, iterated on DMMA blocks), chosen per clique and run concurrently;
- the block-eliminated affine projection (symmetric half-pass SpMVs over SELL-C-σ / Row-SELL layouts, the cached m×m Schur solve, and the rank-one τ correction);
- a fused over-relaxed primal/dual update with residual and certificate reductions.

Cliques are sharded across 1–8 GPUs, and their overlaps are combined with NCCL over NVLink. Results are parity-checked against the reference CPU implementation on five seeded synthetic SDPs. Performance is reported as ADMM iterations/s, time-to-1e-4, and per-kernel fractions of the measured HBM and fp64 rooflines. See `SURVEY.md` for the blueprint and `BASELINE.md` for the baseline plan.

## Status (round 2)

On one B200, config 4 of `BASELINE.json` (400 cliques of order 80, m = 1000, 38 M nonzeros in A), measured by `bench.py` (`profiles/r02/bench_r02.json`):

- **@VALUE@ ADMM iterations/s** with device-resident data under the driver's command (`--steps 20 --warmup 5`, i.e. iterations 6–25, 14 of which still run the cold eigensolver). Round 1 measured 881 there. The steady state after iteration ~20 is about 1,700 iterations/s.
- The default solve reaches 1e-4 in 40 iterations; its loop takes @LOOPMS@ ms (**@TOTOL@ iterations/s**; the reference's loop takes 607 s).
- **End to end** through `solve_decomposed` on host data (H2D copies, device setup, the solve, the report): **@E2E@ iterations/s** (@E2EWALL@ s wall, median of three solves). From the reference's own input layout (dense c over n², A over n² columns) the same call takes @E2EREFWALL@ s.
- The reference algorithm's CPU port on the box's 16 host cores runs at about @REF@ iterations/s.
- The dominant kernel (`k_cone_split`, the warm PSD projection on fp64 DMMA) runs at 18–19% of the measured fp64 DGEMM peak in steady state; the streaming kernels at 58–72% of the measured HBM bandwidth (ncu durations). `DESIGN.md` §3 and §7 say what bounds each, and §8 lists what the round-1 review asked for and what is still open.

Smaller configs 0–3 run at @C0@ / @C1@ / @C2@ / @C3@ iterations/s. All five reproduce the reference's status, iteration count (±2), objectives (1e-6) and iterates (1e-8) — 65 GPU tests and 50 CPU tests.

`profiles/r02/` has the bench lines, ncu launch lists for configs 0–4, `--set full` summaries and counters for the hot kernels and the cold eigensolver, and the phase clocks.

Build with `python -c "import __graft_entry__ as g; g.build()"`. Test with `pytest tests -m "not gpu"` (CPU) and `pytest tests -m gpu` (B200). Benchmark with `python bench.py`. `INTEGRATION.md` describes the C ABI (`include/hsde.h`) and how the reference binds to it.
