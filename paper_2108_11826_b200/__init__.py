"""B200-native pose parsing — drop-in for the reference ``poseflow`` hot path.

The names below mirror ``poseflow`` (``pkg/src/poseflow/__init__.py``) for
the parsing path; ``parse``/``parse_batch`` run on sm_100a kernels through
the C ABI in ``include/pf_b200.h`` (``libpf_b200.so``).  No CPU fallback.
"""

from .core import (
    FeatureMaps,
    Frame,
    HumanPose,
    Keypoint,
    SkeletonTopology,
    TensorF32,
    cell_to_pixel,
    pixel_to_cell,
)
from .errors import (
    BackendError,
    CapacityError,
    ChannelClosed,
    ConfigError,
    ContractError,
    DeviceError,
    FormatError,
    GraphError,
    PipelineError,
    PoseflowError,
)
from .hpt import read_ppm, read_ppm_u8, read_tensor, write_ppm, write_tensor
from .parser import BatchResult, PafParser, ParserParams, PoseSlots, parse, parse_arrays, parse_batch
from .pipeline_ops import (
    OperatorSpec,
    Packet,
    bilinear_resize,
    hwc_to_chw,
    make_batched_postprocess,
    make_postprocess,
    make_preprocess,
    pose_record,
    preprocess_batch,
    resize_planes,
)
from .overlay import OverlayStyle, part_color, visualize, visualize_batch
from .sharding import MultiDeviceParser, ShardedResult
from .skeleton import load_topology, parse_topology
from .producer import render_maps_gpu

__version__ = "0.1.0"

__all__ = [name for name in dir() if not name.startswith("_")]
