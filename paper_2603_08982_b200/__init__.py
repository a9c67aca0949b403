"""SVG-EAR attention for NVIDIA B200 (sm_100a): error-aware routed block-sparse attention with
centroid compensation, as hand-written CUDA behind a C ABI (include/svgear.h).

Public surface mirrors the hot-path part of the reference package `routedattn`:
    prepare, build_error_table, route_error_aware, sparse_attend  (the four-call composition)
and adds the fused operator `svg_ear_attention`, head-parallel sharding helpers, and the callers
either side of the path (SURVEY §8 "next" rows): `schedule` (dense warm-up + warm-started k-means
across denoising steps), `dit` (QKV prologue / attention block), `tensorio` + `config` + `cli`
(QKVT container and the run / sweep / verify harness).
"""

from ._lib import SvgEarError, build_library, lib as load_library
from ._tensors import ShapeError
from .analysis import Prepared, build_error_table, prepare
from .attention import (AttentionResult, FlopCounters, compensation_flops, exact_block_flops,
                        sparse_attend)
from .clustering import (ClusterModel, cluster_means, device_start, inverse_permute_rows, kmeans, kmeans_pp_init,
                         permute_rows, reference_start, seeded_start, segment_means, strided_start)
from .estimator import (BlockErrorTable, estimate_errors, estimate_errors_streaming,
                        estimate_errors_value_aware)
from .operator import operator_workspace_bytes, reference_init, svg_ear_attention
from .router import (FILL_REMAINDER, STOP_AT_FIRST_OVERFLOW, BlockMask, DensityBudget,
                     entry_capacity, mask_from_selected, relaxed_objective, route_error_aware,
                     route_error_aware_entries, route_score, score_top_p)
from .sharding import gather_heads, head_range, sharded_svg_ear_attention
from .schedule import SvgEarStack, WarmupSchedule
from .dit import SvgEarSelfAttention, heads_to_tokens, qkv_prologue, rope_table_3d
from .tensorio import TensorFormatError, read_tensor_file, write_tensor_file
from .config import ConfigError, RunConfig, apply_preset

__version__ = "0.1.0"
