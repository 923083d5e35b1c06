"""paper_2406_16282_b200 -- B200 (sm_100a) hot path of Approx-BP and
Memory-Sharing BP (arXiv 2406.16282): ReGELU2 / ReSiLU2 and MS-LN / MS-RMSNorm.

The compute lives in liblmbp.so (CUDA kernels behind the C ABI of
include/lmbp.h).  This package is the thin Python binding: ``ops`` (same names
as the C ABI), ``modules`` (autograd functions / nn.Modules).  There is no CPU
fallback.
"""
from .ops import (codes_bytes, msln_bwd, msln_fwd, msrms_bwd, msrms_fwd, regelu2_bwd, regelu2_fwd,  # noqa: F401
                  resilu2_bwd, resilu2_fwd, reswiglu2_bwd, reswiglu2_fwd, step_table, stepact_fwd, stepact_bwd,
                  codes_bytes_k, msln_fwd_mixed, msln_bwd_mixed, msrms_fwd_mixed, msrms_bwd_mixed)
from .modules import (MSLayerNorm, MSLayerNormFn, MSRMSNorm, MSRMSNormFn, ReGELU2, ReGELU2Fn, ReSiLU2,  # noqa: F401
                      ReSiLU2Fn, ReSwiGLU2, ReSwiGLU2Fn, saved_bytes)

__all__ = ["regelu2_fwd", "regelu2_bwd", "resilu2_fwd", "resilu2_bwd", "msln_fwd", "msln_bwd", "msrms_fwd",
           "msrms_bwd", "reswiglu2_fwd", "reswiglu2_bwd", "stepact_fwd", "stepact_bwd", "codes_bytes_k", "codes_bytes", "step_table",
           "msln_fwd_mixed", "msln_bwd_mixed", "msrms_fwd_mixed", "msrms_bwd_mixed", "ReGELU2", "ReSiLU2",
           "ReSwiGLU2", "MSLayerNorm", "MSRMSNorm", "ReGELU2Fn", "ReSiLU2Fn", "ReSwiGLU2Fn", "MSLayerNormFn",
           "MSRMSNormFn", "saved_bytes"]
