"""B200-native parallel-in-time Newton ODE solver (hot path of arXiv 2511.01465).

Public names follow the reference package `odescan` (pkg/src/odescan/__init__.py)
for the solver path, so `import paper_2511_01465_b200 as odescan` is a drop-in
for solve()-based code.  All compute runs in libodescan_b200.so (CUDA, sm_100a);
importing this package does not load it — the first solve() does, and fails
loudly if it is missing.
"""

from .baselines import (InnerNewtonFailedError, PararealConfig, PararealResult,
                        solve_parareal, solve_sequential_batch, solve_sequential_explicit,
                        solve_sequential_implicit)
from .affine_scan import (AffineElement, combine, extract_states, identity, init_elements,
                          scan_parallel, scan_sequential)
from .linalg_small import SingularMatrixError, inf_norm, lu_solve, mat_mul, mat_vec
from .newton_pint import (GUESS_POLICIES, BatchSolveReport, NewtonConfig, NonFiniteError,
                          SingularDiagonalBlockError, SolveReport, Trajectory,
                          dense_jacobian_explicit, dense_jacobian_implicit, initial_guess,
                          initial_guess_device, n_steps_for, newton_step_explicit,
                          newton_step_implicit, residual_explicit, residual_implicit, solve,
                          solve_batch)
from .problems import (EXTRA_PROBLEM_NAMES, PROBLEM_NAMES, OdeProblem, allen_cahn, cart_pole,
                       dahlquist, get_problem, logistic, lorenz63, robertson, van_der_pol)
from .steppers import (EULER_TABLEAU, RK4_TABLEAU, STEPPER_NAMES, ButcherTableau,
                       StepperIncrement, explicit_euler, explicit_rk, get_stepper,
                       implicit_euler, trapezoidal)
from .threads import hardware_threads, max_threads, set_threads

__version__ = "0.1.0"

__all__ = [
    "InnerNewtonFailedError", "solve_sequential_explicit", "solve_sequential_implicit",
    "solve_sequential_batch", "PararealConfig", "PararealResult", "solve_parareal",
    "AffineElement", "combine", "identity", "init_elements", "scan_parallel",
    "scan_sequential", "extract_states", "GUESS_POLICIES", "NewtonConfig", "NonFiniteError",
    "SingularDiagonalBlockError", "SolveReport", "BatchSolveReport", "Trajectory",
    "initial_guess", "initial_guess_device", "n_steps_for", "solve", "solve_batch", "PROBLEM_NAMES",
    "EXTRA_PROBLEM_NAMES", "OdeProblem", "cart_pole", "dahlquist", "get_problem", "logistic",
    "robertson", "van_der_pol", "lorenz63", "allen_cahn", "EULER_TABLEAU", "RK4_TABLEAU",
    "STEPPER_NAMES", "ButcherTableau", "StepperIncrement", "explicit_euler", "explicit_rk",
    "get_stepper", "implicit_euler", "trapezoidal", "SingularMatrixError", "inf_norm",
    "lu_solve", "mat_mul", "mat_vec", "hardware_threads", "max_threads", "set_threads",
    "residual_explicit", "residual_implicit", "newton_step_explicit", "newton_step_implicit",
    "dense_jacobian_explicit", "dense_jacobian_implicit", "__version__",
]
