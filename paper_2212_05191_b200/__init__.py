"""paper_2212_05191_b200 -- B200-native SMILE bi-level MoE layer (arXiv 2212.05191).

The product is the C-ABI library ``libsmile.so`` (``include/smile.h``) built from
``csrc/`` for sm_100a; ``smile.py`` is its thin ctypes binding (argument marshalling
only -- every step of the layer runs in the library's CUDA kernels / NCCL calls).
There is no CPU fallback: importing the binding without the built library raises.
"""
from .smile import SmileLayer, SmileError, lib, plan, group, capacity, forward_chunked  # noqa: F401
