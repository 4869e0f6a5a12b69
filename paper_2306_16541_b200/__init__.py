"""freeview-b200: sm_100a implementation of the per-ray-sample path of arXiv 2306.16541.

Public API (mirrors the reference ``freeview`` package and its SPEC):
  render.render_image / Renderer / RenderSettings
  render.skeleton_warp / warp_point / query_radiance / composite / stratified_sample
  model.FreeviewModel                                  the "nets"
  train.train(dataset, config) / Trainer / TrainConfig S:505-513 (patch training)
  autodiff.sample_bone_channels / posenc / transmittance / softmax0 / linear /
           AdamState / adam_step                       ad:403-912 (torch.autograd, CUDA fwd+bwd)
  fused.FusedMlp / fused_forward / naive_forward       fu:64-193
"""

__version__ = "0.1.0"

from .errors import BenchmarkGateError, DimensionError, TrainingError  # noqa: F401
