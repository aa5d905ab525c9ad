"""Seeded synthetic scenes for the BASELINE.json configs (host-side input synthesis).

The paper's test images are not distributed, so every
benchmark and parity case uses this deterministic generator instead: 64-site
Voronoi piecewise-constant regions with intensities U[0, 255], plus a smooth
sinusoid gradient of amplitude 30 (seeded frequency, orientation, phase), plus
i.i.d. N(0, 8^2) texture, clipped to [0, 255].  It runs once per image on the
host, like the reference's own ``synthetic_image`` / ``degrade``
(``imaging.py:207-270``), and feeds bit-identical inputs to the GPU path and
to the CPU oracle.
"""

from __future__ import annotations

import numpy as np


def voronoi_scene(seed: int, height: int, width: int | None = None, n_sites: int = 64,
                  amplitude: float = 30.0, texture: float = 8.0) -> np.ndarray:
    width = height if width is None else width
    gen = np.random.Generator(np.random.PCG64(seed))
    sy = gen.random(n_sites) * height
    sx = gen.random(n_sites) * width
    levels = gen.uniform(0.0, 255.0, n_sites)
    theta = gen.uniform(0.0, 2.0 * np.pi)
    freq = gen.uniform(0.5, 2.0)
    phase = gen.uniform(0.0, 2.0 * np.pi)
    noise = gen.standard_normal((height, width))

    ii = np.arange(height, dtype=np.float64)[:, None]
    jj = np.arange(width, dtype=np.float64)[None, :]
    best = np.full((height, width), np.inf)
    label = np.zeros((height, width), dtype=np.int64)
    for s in range(n_sites):
        d2 = (ii - sy[s]) ** 2 + (jj - sx[s]) ** 2
        closer = d2 < best
        best[closer] = d2[closer]
        label[closer] = s
    u = jj / max(width, 1)
    v = ii / max(height, 1)
    ramp = amplitude * np.sin(2.0 * np.pi * freq * (np.cos(theta) * u + np.sin(theta) * v) + phase)
    img = levels[label] + ramp + texture * noise
    return np.clip(img, 0.0, 255.0)


def voronoi_batch(seeds, height: int, width: int | None = None) -> np.ndarray:
    return np.stack([voronoi_scene(int(s), height, width) for s in seeds])
