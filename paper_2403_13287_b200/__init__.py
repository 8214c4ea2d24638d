"""B200-native LSKUM meshfree Euler solver (drop-in for the reference C ABI).

The product is ``liblskum_b200.so`` (C++ host + CUDA sm_100a engine, sources in
``csrc/``); ``lskum`` is its Python mirror.  See DESIGN.md.
"""
from . import lskum  # noqa: F401
from .lskum import (Cloud, Config, LskumError, Result, Session, run, run_fixed_point)  # noqa: F401

__all__ = ["lskum", "Cloud", "Config", "LskumError", "Result", "Session", "run", "run_fixed_point"]
