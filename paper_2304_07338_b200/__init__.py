"""B200-native photon-field render hot path (arXiv 2304.07338).

The product is the sm_100a C-ABI library libpfgpu.so (include/pf_gpu.h);
this package is its Python host mirror of the reference's pf:: API.
"""
from .api import (AdamConfig, Context, FieldConfig, HashGrid, PathTraceConfig, RenderConfig,  # noqa: F401
                  TraceConfig, TraceResult, TrainConfig, TrainResult, checkpoint_training_state, load_checkpoint, lr_at,
                  save_checkpoint, schedule_radius)
from .scene import (CameraSpec, default_lights, load_photon_map, load_volume,  # noqa: F401
                    save_photon_map, save_volume, synth_photons, synth_volume, tf_scene_a,
                    tf_scene_b)

__all__ = ["AdamConfig", "TrainConfig", "TrainResult", "Context", "FieldConfig", "HashGrid", "PathTraceConfig", "RenderConfig", "TraceConfig", "TraceResult", "schedule_radius", "CameraSpec",
           "default_lights", "synth_volume", "synth_photons", "tf_scene_a", "tf_scene_b",
           "load_volume", "save_volume", "load_photon_map", "save_photon_map"]
