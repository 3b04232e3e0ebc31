"""Pinhole cameras (OpenCV axes: +x right, +y down, +z forward; world +y up).

A camera is 17 float64: c2w row-major 3x4 (12), fx, fy, cx, cy, t_near -- the layout of
``merf_camera`` in include/merf.h and of the oracle's ``cam`` argument.  Poses follow
SURVEY.md section 8(d) (configs C1-C4).
"""
from __future__ import annotations

import math

import numpy as np


def camera_array(c2w: np.ndarray, fx: float, fy: float, cx: float, cy: float,
                 t_near: float = 0.0) -> np.ndarray:
    cam = np.zeros(17, np.float64)
    cam[:12] = np.asarray(c2w, np.float64).reshape(3, 4).ravel()
    cam[12:17] = (fx, fy, cx, cy, t_near)
    return cam


def look_at_camera(pos, target=None, forward=None, W: int = 64, H: int = 64,
                   fov_x_deg: float = 60.0, t_near: float = 0.0) -> np.ndarray:
    pos = np.asarray(pos, np.float64)
    if forward is None:
        forward = np.asarray(target, np.float64) - pos
    f = np.asarray(forward, np.float64)
    f = f / np.linalg.norm(f)
    up = np.array([0.0, 1.0, 0.0])
    r = np.cross(f, up)
    if np.linalg.norm(r) < 1e-9:
        r = np.array([1.0, 0.0, 0.0])
    r = r / np.linalg.norm(r)
    dn = np.cross(f, r)
    c2w = np.zeros((3, 4))
    c2w[:, 0], c2w[:, 1], c2w[:, 2], c2w[:, 3] = r, dn, f, pos
    fx = (W / 2.0) / math.tan(math.radians(fov_x_deg) / 2.0)
    return camera_array(c2w, fx, fx, W / 2.0, H / 2.0, t_near)


def orbit_cameras(n_views: int = 256, W: int = 1920, H: int = 1080, radius: float = 0.9,
                  elevation_deg: float = 15.0, fov_x_deg: float = 60.0,
                  indices=None) -> np.ndarray:
    """C4: views on an orbit around the origin, azimuth k * 360 / n_views."""
    el = math.radians(elevation_deg)
    idx = range(n_views) if indices is None else indices
    cams = []
    for k in idx:
        az = 2.0 * math.pi * k / n_views
        pos = (radius * math.cos(el) * math.cos(az), radius * math.sin(el),
               radius * math.cos(el) * math.sin(az))
        cams.append(look_at_camera(pos, target=(0.0, 0.0, 0.0), W=W, H=H, fov_x_deg=fov_x_deg))
    return np.stack(cams)


def config_cameras(config: str):
    """(cams [n,17], W, H) for a named config."""
    if config == "c1":
        return look_at_camera((0.1, 0.05, -0.2), forward=(0.0, 0.0, 1.0), W=64, H=64)[None], 64, 64
    if config == "c2":
        return look_at_camera((0.3, 0.1, -0.7), target=(0, 0, 0), W=1280, H=720)[None], 1280, 720
    if config == "c3":
        a = look_at_camera((0.95, 0.1, 0.0), forward=(1.0, 0.2, 1.0), W=1920, H=1080)
        b = look_at_camera((3.0, 1.5, 2.0), target=(0, 0, 0), W=1920, H=1080)
        return np.stack([a, b]), 1920, 1080
    if config == "c4":
        return orbit_cameras(256), 1920, 1080
    raise ValueError(config)
