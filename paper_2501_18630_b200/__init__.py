"""paper_2501_18630_b200: B200-native tile rasterizer for Deformable Beta Splatting.

Drop-in for the hot path of the reference package ``betasplat`` (arXiv 2501.18630):
projection -> SH colour -> depth sort + tile binning -> forward raster -> backward, as
hand-written sm_100a kernels in ``libbsr.so`` behind the C-ABI of include/bsr.h.
Names follow betasplat/__init__.py.
"""

__version__ = "0.1.0"

from .camera import Camera  # noqa: F401
from .primitive import GradientBuffer, PrimitiveSet  # noqa: F401
from .rasterizer import (RenderOutput, rasterize, render_backward, render_masked,  # noqa: F401
                         render_tiled)
from .scenes import SplatScene, make_workload  # noqa: F401
