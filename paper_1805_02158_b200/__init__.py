"""B200-native RED fixed-point solver with MPE/RRE/SVD-MPE vector extrapolation.

Drop-in for the reference package ``redve`` (/root/reference/pkg/src/redve,
``__init__.py:18-77``): same names, constructors, argument meaning and
exceptions.  The arithmetic runs in ``libredve_b200.so`` (hand-written
sm_100a CUDA behind the C ABI in ``include/redve_b200.h``); there is no CPU
fallback.  ``RedBatch`` / ``solve_batch`` add the batched device API.
"""

from .batch import RedBatch, solve_batch
from .denoisers import (BUILTIN_DENOISERS, FilterBank, GaussianFilter, Identity, Median3,
                        NotLinear, PatchWeighted, denoise, materialize_dense)
from .errors import (CgNoConvergence, DegenerateSum, InvalidSize, KernelTooLarge, NoConvergence,
                     NonFiniteIterate, RankDeficient, ShapeMismatch, ZeroFirstColumn)
from .extrapolation import (METHODS, MPE, RRE, SVDMPE, ExtrapolationResult, ExtrapolationWeights,
                            QrFactorization, ReconstructionCoefficients, VectorSequenceWindow,
                            build_difference_matrix, extrapolate_batch, extrapolate_once,
                            gamma_mpe, gamma_rre, gamma_svdmpe, mgs_qr, reconstruct,
                            reconstruction_coefficients, small_svd)
from .imaging import (Blur, BlurDownsample, Psf, as_image, convolve_circular, degrade, dft2,
                      embed_psf, gaussian_noise, idft2, make_psf, psf_spectrum, psnr,
                      synthetic_image)
from .pipeline import solve_stream
from .objective import (RedObjective, as_fixed_point_problem, check_local_homogeneity,
                        check_passivity, default_step_size)
from .solvers import (FixedPointProblem, IterationTrace, LinearFixedPointProblem, SolveConfig,
                      Termination, TraceRecord, check_termination, run_fixed_point, run_nesterov,
                      run_steepest_descent, run_ve_cycling, solve)

__version__ = "0.1.0"
