"""B200-native FastMDP-GPU hot path (arXiv 2008.03518): C-ABI library libfmdp.so + binding.

The compute path is libfmdp.so (paper_2008_03518_b200/csrc, sm_100a); this package only
marshals arguments (``fmdp.FMDP``).  See include/fmdp.h and DESIGN.md.
"""
from .build import LIB, build  # noqa: F401


def __getattr__(name):
    if name in ("FMDP", "FmdpError", "ScheduleResult", "lib"):
        from . import fmdp
        return getattr(fmdp, name)
    raise AttributeError(name)
