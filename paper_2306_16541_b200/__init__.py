"""freeview-b200: sm_100a implementation of the per-ray-sample path of arXiv 2306.16541.

Public API (mirrors the reference ``freeview`` package and its SPEC):
  render.render_image / Renderer / RenderSettings
  render.skeleton_warp / warp_point / query_radiance / composite
  model.FreeviewModel                                  the "nets"
  train.Trainer                                        S:505-513 (patch training step)
  ops.sample_bone_channels / posenc / transmittance / adam_step / fused_forward
"""

__version__ = "0.1.0"

from .errors import BenchmarkGateError, DimensionError, TrainingError  # noqa: F401
