"""B200-native (sm_100a) MoE-layer hot path of Compass-v3 (arXiv 2509.09121).

The product is the C-ABI library ``libcompass_moe.so`` (include/compass_moe.h) built from
``csrc/``; this package is its host-side mirror of the reference's SPEC operator interface.
"""
from ._lib import MoEConfigError, MoEError, build, lib  # noqa: F401

__all__ = ["MoEConfigError", "MoEError", "build", "lib", "MoELayer", "MoEConfig", "RouterDecision"]


def __getattr__(name):
    if name in ("MoELayer", "MoEConfig", "RouterDecision"):
        from . import moe
        return getattr(moe, name)
    raise AttributeError(name)
