"""B200-native (sm_100a) GaussianPile slice renderer: the focus-aware slice
renderer, its backward pass, the photometric loss, the fused Adam update and
the 3-D voxelizer of arXiv 2603.20611, behind the reference's API.

The compute path is the in-tree C-ABI library ``_lib/libgpile_b200.so``
(include/gpile_b200.h); importing the API without it raises ImportError.
"""
from .api import *  # noqa: F401,F403
from .api import __all__  # noqa: F401

__version__ = "0.1.0"
