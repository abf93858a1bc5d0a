"""Flow-stage host pieces: the picked-velocity container and the pick gains.

The per-pixel flow arithmetic itself (DC suppression, Hann, power,
autocorrelation, smoothing, argmax: /root/reference/pkg/src/clutterwhiten/
flow.py:51-191, _kernels.py:167-302) runs inside the fused device kernel
(csrc/cw_frame.cuh phases B-E); this module only keeps the reference's
public types and the constant tables the kernel folds in.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .params import FilterParams

__all__ = ["VelocityField", "pick_gains"]


@dataclass
class VelocityField:
    """Per-anchor picked velocity (flow.py:134-144): ``indices[y, x] =
    (ix, iy)`` int32 into the lag grids and ``velocities[y, x] = (vx, vy)``
    float64 in px/frame (velocity == lag at one frame of temporal lag)."""

    indices: np.ndarray
    velocities: np.ndarray


def pick_gains(params: FilterParams) -> tuple[np.ndarray, np.ndarray]:
    """Taper-envelope compensation A(0)/A(l), A(l) = 1/4 + cos(2 pi l / M)/8
    per spatial axis (flow.py:147-163)."""
    out = []
    for grid, m_len in ((params.lag_grid_x, params.mx), (params.lag_grid_y, params.my)):
        lags = np.asarray(grid, dtype=np.float64)
        out.append(0.375 / (0.25 + 0.125 * np.cos(2.0 * np.pi * lags / m_len)))
    return out[0], out[1]
