"""B200-native range-separated (RS) tensor summation of N-particle potentials.

Drop-in for the RS assembly / evaluation path of the reference package
``rstensor`` 0.1.0 (``pkg/src/rstensor/__init__.py:4-94``): same public names,
argument meanings and exception classes.  The host prologue (quadrature,
doubled-grid table, split, support radius) is a bit-exact numpy restatement;
everything per particle system runs in hand-written sm_100a CUDA kernels
behind the C ABI in ``include/rs_b200.h`` (``librsb200.so``).  There is no CPU
fallback for the device path.
"""

from .assembly import (AssemblyConfig, AssemblyResult, DeviceIndexedSystem, DeviceParticles,
                       RSPlan, assemble_long, assemble_short, build_rs, plan_for, reference_for,
                       snap_device, window_slice)
from .errors import (CapabilityError, CapacityError, ConfigError, DomainError, NumericalError,
                     PackingError, ParseError, ResolutionError, RsTensorError, SeparationError,
                     SingularityError, SolverError)
from .formats import (CCT, MAX_DENSE_ELEMENTS, CanonicalTensor, RSCanonical, RSTucker,
                      StorageReport, TuckerTensor, assemble_grid, dense_cct, dense_rs,
                      eval_canonical, eval_canonical_many, eval_cct, eval_rs, eval_rs_many,
                      eval_tucker, eval_tucker_many, lookup_short, storage_report)
from .observables import (EnergyReport, ForceVector, direct_energy, direct_force, force_fd,
                          forces_fd, forces_fd_scale, grad_long, particle_potentials, reference_energy, rs_energy)
from .particles import (Box3, Grid3, IndexedParticleSystem, ParticleSystem, generate_lattice,
                        generate_random_cluster, load_particles, save_particles,
                        separation_distance, snap_to_grid)
from .quadrature import (DEFAULT_R_RANGE, QuadratureRule, RadialKernel, ReferenceCanonical,
                         build_quadrature, effective_support, eval_expansion, project_kernel,
                         split_rank, split_tensor)
from .rankred import (ReductionConfig, SvdSpectrum, c2t_als, rhosvd, rhosvd_error_bound,
                      side_svd, tucker_to_canonical)

__version__ = "0.1.0"
