"""B200-native SUPRA receive-beamforming hot path (arXiv 1711.06127).

DAS beamforming -> fused IQ envelope + log compression -> scan conversion,
as hand-written sm_100a CUDA behind the C ABI in ``include/supra_bf.h``
(``libsupra_bf.so``).  This package is the thin Python binding plus the
multi-GPU driver; it never imports the oracle and has no CPU fallback.
"""
from .binding import (ABI_VERSION, EXPORTS, LIB_PATH, Config, SupraBF, SupraError, lib,
                      make_config)

__all__ = ["ABI_VERSION", "EXPORTS", "LIB_PATH", "Config", "SupraBF", "SupraError", "lib",
           "make_config"]
