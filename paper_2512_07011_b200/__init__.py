"""B200-native Block-Sparse FlashAttention (arXiv 2512.07011), sm_100a.

Drop-in for the reference ``bsfa`` package's hot path: ``flash_forward`` with
Threshold/Dense/FrontierOnly (and the paper's sliding-window / running-max
baseline) gates, ``calibrate`` / ``collect_block_maxima``,
and the ``ThresholdTensor`` file format -- executed by hand-written tcgen05 /
TMA kernels behind the C ABI in ``include/bsfa_b200.h``.  ``attention`` is the
batched GQA entry point on CUDA tensors.
"""

from .errors import (BsfaError, ConfigurationError, DegenerateRowError, FormatError,
                     InvalidInputError, NumericError)
from .tiling import (TileConfig, frontier_blocks, frontier_count, kernel_len, kernel_supports,
                     off_frontier_count)
from .thresholds import ThresholdTensor, load_thresholds, save_thresholds, threshold_lookup
from .gates import (DenseGate, FrontierOnlyGate, GateContext, RunningMaxGate, SlidingWindowGate,
                    ThresholdGate, dense_gate, frontier_only_gate, threshold_gate)
from .core import AttentionOutput, BlockMask, HeadInput
from .trace import FRONTIER, KEPT, SKIPPED, UNREACHABLE, GateTrace
from .attention import AttentionResult, BsfaPlan, attention, flash_forward, reference_scale
from .calibration import (BlockMaximaProfile, CalibrationDiagnostics, CalibrationDump,
                          CalibrationSample, Calibrator, calibrate, collect_block_maxima)
from .dump import MANIFEST_NAME, load_dump, save_dump, write_model_dump
from . import ops  # noqa: F401  (registers torch.ops.bsfa.*)

__version__ = "0.1.0"
