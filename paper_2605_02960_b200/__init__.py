"""B200-native AsyncEP MoE-layer hot path (arxiv/paper_2605_02960, S6.2).

The product is the C-ABI library ``libasyncep.so`` (``include/asyncep.h``); this
package holds its CUDA sources (``csrc/``), the in-tree build (``build.py``), the thin
ctypes binding (``asyncep.py``) and the host-side stack driver (``stack.py``).
"""
from .asyncep import *  # noqa: F401,F403
