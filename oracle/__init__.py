"""fp64 CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct NumPy implementation of what the batched pose-graph
Gauss-Newton / Levenberg-Marquardt hot path computes (Eq. 1 :54-59, GN/LM
and retraction :64, Lie closed forms :157, relative-pose error :479, linear-solve
gradients :224, Eq. 3 / Prop. 1 :243-257 and App. :870-894): dense n x n assembly,
textbook dense Cholesky, step-by-step GN/LM in the paper's order, implicit backward.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  It shares no code with the CUDA
path (``paper_2207_09442_b200/``) and never imports it; the product path never
imports this package.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``): Exp vs scipy expm, Jr closed form vs
the ad-series, coefficient functions vs mpmath, Jacobians vs central finite
differences, App. B curve fit (v0=1 -> v1=3), GN one-step exactness on affine
residuals, hand 2x2 Cholesky/solve examples, brute force vs
scipy.optimize.least_squares on tiny graphs, implicit gradient vs finite differences
of the solve, zero-noise invariants, SE2-in-SE3 embedding, gauge invariance; DLM
(oracle/dlm.py) closed form and eps -> 0 limit; Welsch (oracle/robust.py) SPEC values and
finite differences; Dogleg (nls.dogleg) SPEC hand geometry and GN limit.
Parity unpinned (self-consistency only): the LM damping schedule constants (our
choice, SPEC.md:415 values) and the Dogleg radius constants -- see DESIGN.md "Readings".
"""
from . import lie, costs, linalg, robust, nls, implicit, dlm, unroll  # noqa: F401
