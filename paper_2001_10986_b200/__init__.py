"""B200-native entropic domain decomposition for optimal transport (arXiv 2001.10986).

The hot path (Algorithm 2 sweeps, the coarse-to-fine driver) lives in the
CUDA library libdd_gpu.so behind the C-ABI include/dd.h; this package is the
thin Python binding over it.  It never imports the test oracle.
"""
from .dd import DD, NotConverged, build_schedule, measure_mufu_peak, lib, SO_PATH  # noqa: F401
from .dd import SCHED_FIXED, SCHED_LADDER  # noqa: F401
