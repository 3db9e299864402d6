"""paper_2401_10241_b200 — B200-native Zero Bubble Pipeline Parallelism hot path.

The product is the C-ABI library libzb.so (include/zb.h): tcgen05/TMA GEMMs
for the F, B and W contractions, flash attention, LayerNorm / GeLU /
cross-entropy kernels, the stash-slot stage runtime, the schedulers and the
post-validated AdamW.  This package is the thin Python binding (argument
marshalling; torch is used for device memory and streams only).
"""
from ._lib import ZbError, check, lib  # noqa: F401  (raises ImportError if libzb.so is missing)
from . import api  # noqa: F401
