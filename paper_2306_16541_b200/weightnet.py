"""Canonical weight-volume generator (SPEC ``WeightVolumeNet``, ``S:291-294``; Eq 10, ``P:166``):
a trainable 256-d latent z -> fully-connected layer -> reshape to a 1^3 volume -> five
transposed 3-D convolutions (k = 4, stride 2, padding 1: 1 -> 2 -> 4 -> 8 -> 16 -> 32) ->
logits of the K+1 channel softmax W^c (32^3 x 25 at K = 24).

SURVEY §8f rank 3: one small generator pass per training step (~0.5 GFLOP forward), not on
the per-sample path, so it runs on cuDNN through torch; its layer is pinned to the
reference's own ``conv_transpose3d`` (``ad:633-699``) by golden vectors (``ct_*``).  The
channel widths and the LeakyReLU(0.2) activations are builder-defined (the SPEC cites the
supplementary Fig 6, which gives only the input and output sizes).

With a generator attached, ``Trainer`` writes its output into the model's ``vol_logits``
block before every forward and back-propagates the logits gradient that
``fv_softmax0_bwd`` produces into the generator (instead of updating the logits directly).
"""

from __future__ import annotations

from typing import Sequence

import numpy as np
import torch

LATENT = 256
WIDTHS = (256, 128, 64, 32, 16)


class WeightVolumeNet(torch.nn.Module):
    def __init__(self, n_channels: int = 25, latent: int = LATENT, widths: Sequence[int] = WIDTHS, seed: int = 0):
        super().__init__()
        g = torch.Generator().manual_seed(seed)
        self.z = torch.nn.Parameter(torch.randn(latent, generator=g))          # constant latent
        self.fc = torch.nn.Linear(latent, widths[0])
        chans = list(widths) + [n_channels]
        self.convs = torch.nn.ModuleList(
            [torch.nn.ConvTranspose3d(chans[i], chans[i + 1], 4, stride=2, padding=1) for i in range(5)])
        with torch.no_grad():                                                    # seeded Xavier init
            for m in [self.fc, *self.convs]:
                w = m.weight
                fan_in, fan_out = torch.nn.init._calculate_fan_in_and_fan_out(w)
                lim = float(np.sqrt(6.0 / (fan_in + fan_out)))
                w.copy_((torch.rand(w.shape, generator=g) * 2 - 1) * lim)
                m.bias.zero_()

    def forward(self) -> torch.Tensor:
        """Logits (K+1, 32, 32, 32); W^c = softmax over the channel axis (``softmax0``)."""
        h = self.fc(self.z).view(1, -1, 1, 1, 1)
        for i, conv in enumerate(self.convs):
            h = conv(h)
            if i < len(self.convs) - 1:
                h = torch.nn.functional.leaky_relu(h, 0.2)
        return h[0]
