"""B200-native env-side hot path of URBAN-SIM (citywalk reference):
asynchronous scene sampling + the interactive crowd dynamics step.

Host code is Python over the C ABI of ``libcitywalk_b200.so``
(include/citywalk_b200.h); the hot path is hand-written sm_100a CUDA.
There is no CPU fallback.
"""

from ._lib import build, lib  # noqa: F401

__all__ = ["build", "lib", "urbangen", "crowd", "envcore", "errors", "rng"]
