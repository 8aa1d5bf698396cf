"""Particle spawning (host-side setup, outside the timed path).

``sample_box`` restates the reference's stratified-jitter fill
(/root/reference/pkg/src/softmpm/sampling.py:34-62) with the same RNG call
sequence, so a seed yields the same positions as the reference package
(pinned by tests/golden/kinematics.npz).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import SpawnError


@dataclass
class ParticleSpawn:
    positions: np.ndarray
    rest_volume_per_particle: float
    material_id: int


def _check_margin(positions: np.ndarray, grid) -> None:
    if grid is None:
        return
    lo, hi = grid.margin_bounds()
    if (positions < lo).any() or (positions > hi).any():
        raise SpawnError("spawn volume violates the 1.5-cell domain margin")


def _strata(size: np.ndarray, count: int) -> np.ndarray:
    cell = (float(np.prod(size)) / count) ** (1.0 / 3.0)
    s = np.maximum(1, np.round(size / cell).astype(int))
    while int(np.prod(s)) < count:
        s[int(np.argmax(size / s))] += 1
    return s


def sample_box(center, size, count: int, seed: int, material_id: int = 0,
               grid=None) -> ParticleSpawn:
    """Uniform stratified-jitter fill of an axis-aligned box (sampling.py:43-62)."""
    if count <= 0:
        raise SpawnError("count must be positive")
    center = np.asarray(center, dtype=np.float64)
    size = np.asarray(size, dtype=np.float64)
    if not (size > 0).all():
        raise SpawnError(f"box size must be positive, got {size}")
    rng = np.random.default_rng(seed)
    strata = _strata(size, count)
    cells = np.stack(np.unravel_index(np.arange(int(np.prod(strata))), strata), axis=1)
    chosen = cells[rng.permutation(len(cells))[:count]]
    jitter = rng.random((count, 3))
    positions = (center - 0.5 * size) + (chosen + jitter) * (size / strata)
    _check_margin(positions, grid)
    return ParticleSpawn(positions=positions,
                         rest_volume_per_particle=float(np.prod(size)) / count,
                         material_id=material_id)
