"""Pose refinement (SPEC ``refine_pose`` / ``PoseRefinerNet``, ``S:287-290``, ``S:309-317``;
Eqs 5-6, ``P:130-140``) and the differentiable motion bases it trains through.

The skinning warp's backward (``fv_warp_bwd_g``) returns dL/dG_i for the 24 per-frame
motion bases; this module chains it to the joint angles on the host in float64 torch --
24 small matrices per frame, the reference's own Tape path (``sk:186-303``):
  * ``rodrigues`` (series branch for |w|^2 < 1e-8, ``sk:186-209``), forward kinematics
    ``T_i = T_parent o translate(rest_offset_i) o rotate(w_i)`` (``sk:240-273``) and
    ``G_i = T_i(canonical) o T_i(observed)^-1`` (``sk:288-303``), pinned to the reference's
    gradients by golden vectors (``mb_dang``, ``mb_droot``);
  * ``PoseRefinerNet``: an MLP Omega (K*3) -> dOmega with a zero-initialised last layer, and
    ``refine``: w^o_k = log(R(dw_k) R(w_k)) per joint (Eq 6), written as
    ``w + (log(R(dw) R(w)) - log(R(w)))`` so a fresh refiner returns the pose exactly.
Layer widths of the refiner are builder-defined (the SPEC cites supplementary Fig 5).
"""

from __future__ import annotations

from typing import Tuple

import torch

from .skeleton import Skeleton

F64 = torch.float64


def skew(w: torch.Tensor) -> torch.Tensor:
    z = torch.zeros_like(w[:, 0])
    return torch.stack([torch.stack([z, -w[:, 2], w[:, 1]], -1),
                        torch.stack([w[:, 2], z, -w[:, 0]], -1),
                        torch.stack([-w[:, 1], w[:, 0], z], -1)], -2)


def rodrigues(w: torch.Tensor) -> torch.Tensor:
    """(K,3) axis-angle -> (K,3,3); Taylor branch near 0 so map and gradient are exact there."""
    th2 = (w * w).sum(-1)
    near = th2 < 1e-8
    safe = torch.where(near, torch.ones_like(th2), th2)
    th = torch.sqrt(safe)
    a = torch.where(near, 1.0 - th2 / 6.0, torch.sin(th) / th)
    b = torch.where(near, 0.5 - th2 / 24.0, (1.0 - torch.cos(th)) / safe)
    k = skew(w)
    eye = torch.eye(3, dtype=w.dtype, device=w.device).expand(w.shape[0], 3, 3)
    return eye + a[:, None, None] * k + b[:, None, None] * (k @ k)


def rotation_log(r: torch.Tensor) -> torch.Tensor:
    """(K,3,3) rotation -> axis-angle (K,3), angle in [0, pi): theta = atan2(|v|, (tr-1)/2),
    v = vee(R - R^T)/2, w = theta / sin(theta) * v (series near 0)."""
    v = 0.5 * torch.stack([r[:, 2, 1] - r[:, 1, 2], r[:, 0, 2] - r[:, 2, 0], r[:, 1, 0] - r[:, 0, 1]], -1)
    s = torch.sqrt((v * v).sum(-1).clamp_min(1e-300))
    c = 0.5 * (r[:, 0, 0] + r[:, 1, 1] + r[:, 2, 2] - 1.0)
    th = torch.atan2(s, c)
    near = s < 1e-6
    f = torch.where(near, 1.0 + th * th / 6.0, th / torch.where(near, torch.ones_like(s), s))
    return f[:, None] * v


def world_transforms(skel: Skeleton, angles: torch.Tensor, root: torch.Tensor):
    rot = rodrigues(angles)
    k = skel.bone_count
    r_out = [None] * k
    t_out = [None] * k
    offs = torch.as_tensor(skel.rest_offset, dtype=angles.dtype, device=angles.device)
    for i in skel.order():
        p = int(skel.parent[i])
        if p < 0:
            r_out[i] = rot[i]
            t_out[i] = root + offs[i]
        else:
            r_out[i] = r_out[p] @ rot[i]
            t_out[i] = t_out[p] + r_out[p] @ offs[i]
    return torch.stack(r_out), torch.stack(t_out)


def motion_basis(skel: Skeleton, angles: torch.Tensor, root: torch.Tensor) -> Tuple[torch.Tensor, torch.Tensor]:
    """G_r (K,3,3), G_t (K,3): observation -> canonical per bone, differentiable in the pose."""
    with torch.no_grad():
        rc, tc = world_transforms(skel, torch.as_tensor(skel.canonical_angles, dtype=angles.dtype),
                                  torch.as_tensor(skel.canonical_root, dtype=angles.dtype))
    ro, to = world_transforms(skel, angles, root)
    g_r = rc @ ro.transpose(1, 2)
    g_t = tc - (g_r @ to[:, :, None])[:, :, 0]
    return g_r, g_t


class PoseRefinerNet(torch.nn.Module):
    """Omega (K*3) -> dOmega (K*3); zero-initialised last layer."""

    def __init__(self, n_joints: int = 24, width: int = 256, depth: int = 3, seed: int = 0):
        super().__init__()
        g = torch.Generator().manual_seed(seed)
        dims = [3 * n_joints] + [width] * (depth - 1) + [3 * n_joints]
        self.layers = torch.nn.ModuleList([torch.nn.Linear(a, b, dtype=F64) for a, b in zip(dims[:-1], dims[1:])])
        with torch.no_grad():
            for i, m in enumerate(self.layers):
                if i == len(self.layers) - 1:
                    m.weight.zero_()
                    m.bias.zero_()
                else:
                    lim = (6.0 / (m.in_features + m.out_features)) ** 0.5
                    m.weight.copy_((torch.rand(m.weight.shape, generator=g, dtype=F64) * 2 - 1) * lim)
                    m.bias.zero_()

    def forward(self, omega: torch.Tensor) -> torch.Tensor:
        h = omega.reshape(-1)
        for i, m in enumerate(self.layers):
            h = m(h)
            if i < len(self.layers) - 1:
                h = torch.relu(h)
        return h.view(-1, 3)

    def refine(self, omega: torch.Tensor) -> torch.Tensor:
        """w^o_k = log(R(dw_k) R(w_k)) (Eq 6), exact identity for a zero dOmega."""
        d = self(omega)
        r = rodrigues(omega)
        return omega + (rotation_log(rodrigues(d) @ r) - rotation_log(r))
