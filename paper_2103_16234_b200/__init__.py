"""paper_2103_16234_b200 — B200-native fp32 forward convolution (cuConv,
arXiv 2103.16234), a drop-in for convkit's forward-convolution entry point.

Host API (numpy in/out, reference signatures and exceptions):
    conv_twostage, stage1_scalar_prods, stage2_sum, workspace_bytes,
    conv_forward (any stride), conv_forward_layers (pipelined sequence),
    RunStats, PartialSums, DEFAULT_WORKSPACE_LIMIT
Device API (torch CUDA tensors, current stream):
    conv2d, ConvLayer
Shapes, tensors, plans, errors:
    ConvConfig, Tensor4, make_tensor, DeviceModel, LaunchPlan, plan_launch, ...

Compute always runs in the hand-written sm_100a kernels of libb2conv.so
(built by ``python -m paper_2103_16234_b200.build``); there is no CPU path.
"""

from .configs import (BATCH_SIZES, ConvConfig, filter_dims, filter_row_reuse, input_dims, output_dims,
                      parse_config_file, preset_configs, same_padding)
from .errors import (ConvKitError, DeviceError, FormatError, InvalidConfig, InvalidPlan, InvalidShape,
                     ParseError, ShapeMismatch, Unsupported, UnsupportedFilter, WorkspaceExceeded)
from .execmodel import (DeviceModel, LaunchPlan, TilePlan, block_position_ranges, family_names,
                        matching_families, plan_launch, select_tiles, theoretical_reuse, validate_plan)
from .tensor import Tensor4, load_tensor, make_tensor, read_padded, save_tensor
from .twostage import (DEFAULT_WORKSPACE_LIMIT, PartialSums, RunStats, conv_forward, conv_forward_layers,
                       conv_twostage, stage1_scalar_prods, stage2_sum, workspace_bytes)
from .engine import ConvLayer, conv2d

__version__ = "0.1.0"
