"""NEXT-4 oracle: progressive rendering.  TEST INFRASTRUCTURE ONLY.

"the image is first rendered at a lower resolution.  When the camera rests additional low
resolution images are rendered that are dynamically combined into the final high resolution
image ... progressive upsampling speeds up rendering in proportion to the ratio of target
resolution and initial render resolution".

Reading P1: with stride s, pass p in [0, s^2) renders the pixels of the
sub-lattice (s i + p mod s, s j + floor(p / s)) at full-resolution pixel centres (so every
pixel is computed exactly as in the full render, reading D18); the s^2 passes partition the
frame, so "combining" them is interleaving.  The preview of a pass is its nearest
upsampling: rendered pixel (px, py) also colours the block [px, px + s) x [py, py + s),
clipped to the frame.  Colours of rendered pixels come from `oracle.render(..., pixels=)`.
"""
from __future__ import annotations

import numpy as np


def pass_offset(stride: int, pass_: int):
    """(ox, oy) of pass `pass_` (P1)."""
    if not (1 <= stride and 0 <= pass_ < stride * stride):
        raise ValueError("pass must be in [0, stride^2)")
    return pass_ % stride, pass_ // stride


def pass_pixels(W: int, H: int, stride: int, pass_: int) -> np.ndarray:
    """row-major pixel ids y * W + x rendered by the pass, in increasing order."""
    ox, oy = pass_offset(stride, pass_)
    xs = np.arange(ox, W, stride, dtype=np.int64)
    ys = np.arange(oy, H, stride, dtype=np.int64)
    return (ys[:, None] * W + xs[None, :]).ravel()


def fill_source(W: int, H: int, stride: int, pass_: int) -> np.ndarray:
    """for every pixel of the frame, the rendered pixel whose colour the preview shows there
    (nearest upsampling), or -1 where the pass leaves the pixel untouched."""
    ox, oy = pass_offset(stride, pass_)
    src = np.full(W * H, -1, np.int64)
    for y in range(H):
        if y < oy:
            continue
        sy = oy + ((y - oy) // stride) * stride
        for x in range(W):
            if x < ox:
                continue
            sx = ox + ((x - ox) // stride) * stride
            src[y * W + x] = sy * W + sx
    return src
