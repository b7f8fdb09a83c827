"""B200-native semi-implicit RIDC (Ong, Melfi & Christlieb, arXiv:1209.4297).

Drop-in for the reference package's marching path (``ridc.engine``,
``ridc.problems``, ``ridc.quadrature``, ``ridc.studies.integrate_scheme``):
same names and argument meanings, computed by hand-written sm_100a kernels
behind the C-ABI in include/ridc_b200.h.  No CPU fallback.
"""

from .errors import (ConfigError, DeterminismError, DimensionMismatch, NonFiniteStateError,
                     PipelineProtocolError, SingularMatrixError, NewtonConvergenceError,
                     CudaError, SOLVER_FAILURES)
from .quadrature import (MAX_LEVEL, QuadratureWeights, apply_quadrature, startup_weights,
                         steady_weights)
from . import problems
from .engine import (Engine, LevelWindow, RidcConfig, RidcSolution, correct_step,
                     predict_step, restart_partition, run_pipelined, run_serial,
                     startup_delay)
from .studies import integrate_scheme, scheme_levels
from .tableaus import ButcherPair, imex3_tableau, imex4_tableau
from .steppers import ArkEngine, ark_step, fbe_step, integrate_ark

__version__ = "0.1.0"
