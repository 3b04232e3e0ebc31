"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds NONE of the method's arithmetic (no contraction, no traversal, no
interpolation, no decoding, no compositing): it only builds baked-scene arrays and camera
structs from a seed.  See DESIGN.md "Input recipe".
"""
from .scene import (MerfScene, make_scene, constant_scene, random_scene, CONFIGS,
                    pack_bits, unpack_bits)
from .cameras import look_at_camera, config_cameras, orbit_cameras, camera_array

__all__ = ["MerfScene", "make_scene", "constant_scene", "random_scene", "CONFIGS", "pack_bits",
           "unpack_bits", "look_at_camera", "config_cameras", "orbit_cameras", "camera_array"]
