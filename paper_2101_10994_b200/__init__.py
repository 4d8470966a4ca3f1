"""B200-native NGLOD render hot path (arXiv 2101.10994).

A drop-in for the hot-path subset of the reference package `octfield`
(octfield/__init__.py:11-164): octree construction, per-LOD SDF queries,
the breadth-first ray-octree traversal and the sparse sphere tracer with
normals and shading. Every compute entry point runs hand-written sm_100a
CUDA kernels through the C ABI in include/nglod_b200.h; there is no CPU
fallback.
"""

from .errors import (
    ConfigError,
    FormatError,
    OctfieldError,
    SamplingError,
    SceneError,
    StructuralError,
    TrainingDiverged,
)
from .octree import (
    DOMAIN_MAX,
    DOMAIN_MIN,
    Aabb,
    SparseVoxelOctree,
    build_octree,
    locate,
    morton_decode,
    morton_encode,
    ray_aabb_batch,
    storage_bytes,
    voxel_bounds,
)
from .field import (
    FEATURE_DIM,
    HIDDEN_DIM,
    Decoder,
    EvalCounter,
    NeuralField,
    blend,
    decode,
    empty_space_value,
    forward,
    forward_levels,
    new_field,
    predict,
    sum_features,
    trilinear,
    DecoderGrads,
    FieldGradients,
    LevelInterp,
    backward,
    scatter_add_rows,
)
from .sampling import SampleSet, build_epoch_set, surface_points
from .trainer import AdamState, EpochStats, TrainConfig, active_levels_for, adam_step, loss_batch, train
from .modelio import load_model, save_model, serialized_bytes
from .metrics import (
    EvalReport,
    bench_frame,
    chamfer_l1,
    evaluate,
    fibonacci_cameras,
    giou,
    image_metrics,
    sample_predicted_surface,
    surface_accuracy,
)
from .traversal import RayBundle, RayVoxelPairList, exclusive_sum, ray_segments, ray_trace_octree
from .render import (
    Camera,
    FrameBuffer,
    FrameReport,
    RenderConfig,
    RenderSession,
    normals,
    query_field,
    render,
    render_batch,
    render_frames,
    select_lod,
    shade,
    sphere_trace,
    trace_rays,
    write_ppm,
)

__version__ = "0.1.0"

__all__ = [
    "Aabb", "Camera", "ConfigError", "Decoder", "DOMAIN_MAX", "DOMAIN_MIN", "EvalCounter", "FEATURE_DIM",
    "FormatError", "FrameBuffer", "FrameReport", "HIDDEN_DIM", "NeuralField", "OctfieldError", "RayBundle",
    "RayVoxelPairList", "RenderConfig", "RenderSession", "SamplingError", "SceneError", "SparseVoxelOctree",
    "StructuralError", "TrainingDiverged", "blend", "build_octree", "decode", "empty_space_value",
    "exclusive_sum", "forward", "forward_levels", "locate", "morton_decode", "morton_encode", "new_field",
    "normals", "predict", "query_field", "ray_aabb_batch", "ray_segments", "ray_trace_octree", "render",
    "render_batch",
    "render_frames",
    "select_lod", "shade", "sphere_trace", "storage_bytes", "sum_features", "trace_rays", "trilinear",
    "voxel_bounds", "write_ppm", "DecoderGrads", "FieldGradients", "LevelInterp", "backward", "scatter_add_rows",
    "SampleSet", "build_epoch_set", "surface_points", "AdamState", "EpochStats", "TrainConfig",
    "active_levels_for", "adam_step", "loss_batch", "train", "load_model", "save_model", "serialized_bytes",
    "EvalReport", "bench_frame", "chamfer_l1", "evaluate", "fibonacci_cameras", "giou", "image_metrics",
    "sample_predicted_surface", "surface_accuracy",
]
