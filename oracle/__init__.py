"""float64 CPU oracle for the ReGELU2/ReSiLU2 + MS-LN/MS-RMSNorm hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_2406_16282_b200``) never imports it, and it
shares no code, header, table or constant with the CUDA library.

The arithmetic lives in ``oracle.c`` (binary64, scalar loops, OpenMP across
independent rows only).  This wrapper only marshals numpy arrays:

* ``decode``   -- exact conversion of stored fp32 / bf16 / fp16 values to float64
                  (every such value is exactly representable in binary64);
* ``round_to`` -- round-to-nearest-even conversion float64 -> binary32 -> storage
                  type, used only for the bitwise act-backward contract
                  (reading R5) and to hand oracle outputs to the GPU as
                  inputs of a later step.

Storage convention: fp32 -> ``np.float32``; fp16 -> ``np.float16``; bf16 ->
``np.uint16`` holding the raw bf16 bit pattern (numpy has no bfloat16).

Citations follow SURVEY.md: P:L<n> = PAPER.md line n, S:L<n> = SPEC.md line n.
Every function is pinned in tests/test_oracle_pins.py; none is "parity
unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

GELU, SILU = 0, 1
KINDS = {"gelu": GELU, "silu": SILU}
DTYPES = ("f32", "bf16", "f16")


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (-O2, no fast-math, OpenMP)."""
    if (not force and os.path.exists(_LIB_PATH)
            and os.path.getmtime(_LIB_PATH) >= os.path.getmtime(_SRC)):
        return _LIB_PATH
    cmd = ["gcc", "-std=c11", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp",
           "-fPIC", "-shared", _SRC, "-o", _LIB_PATH + ".tmp", "-lm"]
    subprocess.check_call(cmd)
    os.replace(_LIB_PATH + ".tmp", _LIB_PATH)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        d, i64, i32 = ctypes.c_double, ctypes.c_int64, ctypes.c_int
        p = ctypes.c_void_p
        for name in ("oracle_gelu", "oracle_silu", "oracle_gelu_deriv", "oracle_silu_deriv"):
            f = getattr(L, name)
            f.restype, f.argtypes = d, [d]
        L.oracle_combo_eval.restype, L.oracle_combo_eval.argtypes = d, [i32, d]
        L.oracle_step_table.restype, L.oracle_step_table.argtypes = i32, [i32, p, p, p]
        L.oracle_act_fwd.restype, L.oracle_act_fwd.argtypes = i32, [i32, p, i64, p, p, i32]
        L.oracle_act_bwd.restype, L.oracle_act_bwd.argtypes = i32, [i32, p, p, i64, p, i32]
        L.oracle_act_bwd_contract_exact.restype = i32
        L.oracle_act_bwd_contract_exact.argtypes = [i32, p, p, i64, p, i32]
        for name in ("oracle_msln_fwd", "oracle_msrms_fwd"):
            f = getattr(L, name)
            f.restype, f.argtypes = i32, [p, i64, i64, d, p, p, i32]
        for name in ("oracle_msln_bwd", "oracle_msrms_bwd"):
            f = getattr(L, name)
            f.restype, f.argtypes = i32, [p, p, p, i64, i64, p, i32]
        L.oracle_max_threads.restype, L.oracle_max_threads.argtypes = i32, []
        L.oracle_stepact_fwd.restype = i32
        L.oracle_stepact_fwd.argtypes = [i32, i32, p, p, i64, p, p]
        L.oracle_stepact_bwd.restype = i32
        L.oracle_stepact_bwd.argtypes = [i32, p, p, p, i64, p]
        L.oracle_regelu2d_table.restype = i32
        L.oracle_regelu2d_table.argtypes = [p, p]
        L.oracle_reswiglu2_fwd.restype = i32
        L.oracle_reswiglu2_fwd.argtypes = [p, p, i64, p, p, p, i32]
        L.oracle_reswiglu2_bwd.restype = i32
        L.oracle_reswiglu2_bwd.argtypes = [p, p, p, p, i64, p, p, i32]
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def _kind(kind) -> int:
    return KINDS[kind] if isinstance(kind, str) else int(kind)


# Threads the oracle uses when a call does not say (None = OpenMP's default,
# which honours OMP_NUM_THREADS; bench.py sets it to the host's usable cores).
DEFAULT_THREADS = None


def max_threads() -> int:
    if DEFAULT_THREADS is not None:
        return int(DEFAULT_THREADS)
    return int(lib().oracle_max_threads())


def _nt(nthreads):
    return max_threads() if nthreads is None else int(nthreads)


# --------------------------------------------------------------------------
# storage <-> float64 (plumbing; exact in the decode direction)
# --------------------------------------------------------------------------
def decode(a: np.ndarray, dtype: str) -> np.ndarray:
    """Exact float64 value of every stored element."""
    if dtype == "f32":
        return np.ascontiguousarray(a, dtype=np.float32).astype(np.float64)
    if dtype == "f16":
        return np.ascontiguousarray(a, dtype=np.float16).astype(np.float64)
    if dtype == "bf16":
        bits = np.ascontiguousarray(a, dtype=np.uint16).astype(np.uint32) << 16
        with np.errstate(invalid="ignore"):   # NaN payloads
            return bits.view(np.float32).astype(np.float64)
    raise ValueError(dtype)


def _f32_to_bf16_bits(f: np.ndarray) -> np.ndarray:
    """binary32 -> bfloat16 bit pattern, round to nearest, ties to even."""
    u = np.ascontiguousarray(f, dtype=np.float32).view(np.uint32).astype(np.uint64)
    bias = 0x7FFF + ((u >> 16) & 1)
    out = ((u + bias) >> 16).astype(np.uint16)
    nan = np.isnan(np.ascontiguousarray(f, dtype=np.float32))
    out[nan] = ((u[nan] >> 16) | 0x0040).astype(np.uint16)   # quiet NaN, sign kept
    return out


def round_to(v: np.ndarray, dtype: str) -> np.ndarray:
    """float64 -> binary32 (RNE) -> storage type (RNE)."""
    with np.errstate(over="ignore"):
        f = np.ascontiguousarray(v, dtype=np.float64).astype(np.float32)
    if dtype == "f32":
        return f
    if dtype == "f16":
        with np.errstate(over="ignore"):      # overflow to +-inf is the RNE result
            return f.astype(np.float16)
    if dtype == "bf16":
        return _f32_to_bf16_bits(f)
    raise ValueError(dtype)


# --------------------------------------------------------------------------
# Step table and scalar references
# --------------------------------------------------------------------------
def step_table(kind):
    """(c[3], s[4], a[2]) in float64: thresholds, levels, published weights.
    P:L1062-1063 (GELU), P:L1139-1140 (SiLU); levels P:L1017."""
    c = np.zeros(3)
    s = np.zeros(4)
    a = np.zeros(2)
    rc = lib().oracle_step_table(_kind(kind), _ptr(c), _ptr(s), _ptr(a))
    if rc != 0:
        raise ValueError(kind)
    return c, s, a


def gelu(x: float) -> float:
    return lib().oracle_gelu(float(x))


def silu(x: float) -> float:
    return lib().oracle_silu(float(x))


def act(kind, x: float) -> float:
    return gelu(x) if _kind(kind) == GELU else silu(x)


def act_deriv(kind, x: float) -> float:
    L = lib()
    return L.oracle_gelu_deriv(float(x)) if _kind(kind) == GELU else L.oracle_silu_deriv(float(x))


def combo_eval(kind, x: float) -> float:
    """h~_{a*,c*}(x), Eq. 14 / P:L1017."""
    return lib().oracle_combo_eval(_kind(kind), float(x))


def codes_bytes(n: int) -> int:
    """Packed 2-bit codes, four per byte: ceil(n/4) bytes."""
    return (int(n) + 3) // 4


def unpack_codes(codes: np.ndarray, n: int) -> np.ndarray:
    """Element j <- bits 2(j&3) of byte j>>2."""
    codes = np.asarray(codes, dtype=np.uint8)
    j = np.arange(n)
    return ((codes[j >> 2] >> (2 * (j & 3))) & 3).astype(np.uint8)


# --------------------------------------------------------------------------
# Hot-path definitions (fp64)
# --------------------------------------------------------------------------
def act_fwd(kind, x64: np.ndarray, nthreads=None):
    """ReGELU2/ReSiLU2 forward: (y = h(x), packed codes).  P:L413-416."""
    x = np.ascontiguousarray(x64, dtype=np.float64).reshape(-1)
    n = x.size
    y = np.empty(n, dtype=np.float64)
    codes = np.zeros(codes_bytes(n), dtype=np.uint8)
    if n:
        rc = lib().oracle_act_fwd(_kind(kind), _ptr(x), n, _ptr(y), _ptr(codes), _nt(nthreads))
        assert rc == 0
    return y.reshape(np.shape(x64)), codes


def act_bwd(kind, codes: np.ndarray, dy64: np.ndarray, nthreads=None):
    """Value mode: dx = s[code] * dy in fp64.  P:L371."""
    dy = np.ascontiguousarray(dy64, dtype=np.float64).reshape(-1)
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    n = dy.size
    if codes.size != codes_bytes(n):
        raise ValueError("codes/element count mismatch (S:L174)")
    dx = np.empty(n, dtype=np.float64)
    if n:
        rc = lib().oracle_act_bwd(_kind(kind), _ptr(codes), _ptr(dy), n, _ptr(dx), _nt(nthreads))
        assert rc == 0
    return dx.reshape(np.shape(dy64))


def act_bwd_contract(kind, codes: np.ndarray, dy_stored: np.ndarray, dtype: str, nthreads=None):
    """Bitwise contract (reading R5): RN_T(RN32(dy * RN32(s[code]))) in the
    storage type of ``dy_stored``."""
    dy = decode(dy_stored, dtype).reshape(-1)
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    n = dy.size
    if codes.size != codes_bytes(n):
        raise ValueError("codes/element count mismatch (S:L174)")
    prod = np.empty(n, dtype=np.float64)
    if n:
        rc = lib().oracle_act_bwd_contract_exact(_kind(kind), _ptr(codes), _ptr(dy), n,
                                                 _ptr(prod), _nt(nthreads))
        assert rc == 0
    return round_to(prod, dtype).reshape(np.shape(dy_stored))


def _rows(x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    if x.ndim != 2:
        raise ValueError("expected [rows, cols]")
    return x


def msln_fwd(x64, eps: float, nthreads=None):
    """MS-LN forward, Alg. 2: (y, rstd = 1/sigma)."""
    x = _rows(x64)
    R, H = x.shape
    y = np.empty_like(x)
    rstd = np.empty(R)
    if R:
        assert lib().oracle_msln_fwd(_ptr(x), R, H, float(eps), _ptr(y), _ptr(rstd), _nt(nthreads)) == 0
    return y, rstd


def msln_bwd(dy64, y64, rstd64, nthreads=None):
    """MS-LN backward, Alg. 2, from (y, rstd, dy) only."""
    dy, y = _rows(dy64), _rows(y64)
    rstd = np.ascontiguousarray(rstd64, dtype=np.float64).reshape(-1)
    R, H = dy.shape
    if y.shape != dy.shape or rstd.size != R:
        raise ValueError("token/shape mismatch (S:L266)")
    dx = np.empty_like(dy)
    if R:
        assert lib().oracle_msln_bwd(_ptr(dy), _ptr(y), _ptr(rstd), R, H, _ptr(dx), _nt(nthreads)) == 0
    return dx


def msrms_fwd(x64, eps: float, nthreads=None):
    """MS-RMSNorm forward, Alg. 3."""
    x = _rows(x64)
    R, H = x.shape
    y = np.empty_like(x)
    rstd = np.empty(R)
    if R:
        assert lib().oracle_msrms_fwd(_ptr(x), R, H, float(eps), _ptr(y), _ptr(rstd), _nt(nthreads)) == 0
    return y, rstd


def msrms_bwd(dy64, y64, rstd64, nthreads=None):
    """MS-RMSNorm backward, Alg. 3."""
    dy, y = _rows(dy64), _rows(y64)
    rstd = np.ascontiguousarray(rstd64, dtype=np.float64).reshape(-1)
    R, H = dy.shape
    if y.shape != dy.shape or rstd.size != R:
        raise ValueError("token/shape mismatch (S:L266)")
    dx = np.empty_like(dy)
    if R:
        assert lib().oracle_msrms_bwd(_ptr(dy), _ptr(y), _ptr(rstd), R, H, _ptr(dx), _nt(nthreads)) == 0
    return dx


# --------------------------------------------------------------------------
# k-bit step activations
# --------------------------------------------------------------------------
def codes_bytes_k(n: int, k: int) -> int:
    return (int(n) * int(k) + 7) // 8


def regelu2d_table():
    """(c[3], s[4]) of ReGELU2-d, App. I."""
    c, s = np.zeros(3), np.zeros(4)
    lib().oracle_regelu2d_table(_ptr(c), _ptr(s))
    return c, s


def stepact_fwd(kind, k, thresholds, x64):
    x = np.ascontiguousarray(x64, dtype=np.float64).reshape(-1)
    c = np.ascontiguousarray(thresholds, dtype=np.float64)
    if c.size != (1 << k) - 1:
        raise ValueError("need 2^k - 1 thresholds")
    n = x.size
    y = np.empty(n)
    codes = np.zeros(codes_bytes_k(n, k), dtype=np.uint8)
    if n:
        assert lib().oracle_stepact_fwd(_kind(kind), k, _ptr(c), _ptr(x), n, _ptr(y), _ptr(codes)) == 0
    return y.reshape(np.shape(x64)), codes


def stepact_bwd(k, levels, codes, dy64):
    dy = np.ascontiguousarray(dy64, dtype=np.float64).reshape(-1)
    s = np.ascontiguousarray(levels, dtype=np.float64)
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    n = dy.size
    if s.size != (1 << k) or codes.size != codes_bytes_k(n, k):
        raise ValueError("table / codes size")
    dx = np.empty(n)
    if n:
        assert lib().oracle_stepact_bwd(k, _ptr(s), _ptr(codes), _ptr(dy), n, _ptr(dx)) == 0
    return dx.reshape(np.shape(dy64))


def stepact_bwd_contract(k, levels, codes, dy_stored, dtype):
    """RN_T(RN32(dy * RN32(level))) -- the binary32 product is exact in binary64."""
    s32 = np.asarray(levels, dtype=np.float64).astype(np.float32).astype(np.float64)
    prod = stepact_bwd(k, s32, codes, decode(dy_stored, dtype))
    return round_to(prod, dtype).reshape(np.shape(dy_stored))


# --------------------------------------------------------------------------
# ReSwiGLU2: h = SiLU(gate) * up, ReSiLU2 backward
# --------------------------------------------------------------------------
def reswiglu2_fwd(g64, u64, nthreads=None):
    """(h = SiLU(g) u, a = SiLU(g), codes of g) in float64."""
    g = np.ascontiguousarray(g64, dtype=np.float64).reshape(-1)
    u = np.ascontiguousarray(u64, dtype=np.float64).reshape(-1)
    if g.size != u.size:
        raise ValueError("shape mismatch")
    n = g.size
    h, a = np.empty(n), np.empty(n)
    codes = np.zeros(codes_bytes(n), dtype=np.uint8)
    if n:
        assert lib().oracle_reswiglu2_fwd(_ptr(g), _ptr(u), n, _ptr(h), _ptr(a), _ptr(codes), _nt(nthreads)) == 0
    shp = np.shape(g64)
    return h.reshape(shp), a.reshape(shp), codes


def reswiglu2_bwd(dh64, u64, a64, codes, nthreads=None):
    """Value mode: (dg = dh u s[code], du = dh a) in float64."""
    dh = np.ascontiguousarray(dh64, dtype=np.float64).reshape(-1)
    u = np.ascontiguousarray(u64, dtype=np.float64).reshape(-1)
    a = np.ascontiguousarray(a64, dtype=np.float64).reshape(-1)
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    n = dh.size
    if u.size != n or a.size != n or codes.size != codes_bytes(n):
        raise ValueError("shape mismatch")
    dg, du = np.empty(n), np.empty(n)
    if n:
        assert lib().oracle_reswiglu2_bwd(_ptr(dh), _ptr(u), _ptr(a), _ptr(codes), n, _ptr(dg), _ptr(du),
                                          _nt(nthreads)) == 0
    shp = np.shape(dh64)
    return dg.reshape(shp), du.reshape(shp)


def reswiglu2_bwd_contract(dh_st, u_st, a_st, codes, dtype):
    """Bitwise contract of the fused kernel = the unfused composition:
    du = RN_T(RN32(dh a)); da = RN_T(RN32(dh u)); dg = act_bwd_contract(da).
    Products of two binary32 values are exact in binary64."""
    dh, u, a = decode(dh_st, dtype), decode(u_st, dtype), decode(a_st, dtype)
    du = round_to(dh * a, dtype)
    da = round_to(dh * u, dtype)
    dg = act_bwd_contract("silu", codes, da, dtype)
    return dg, du


# --------------------------------------------------------------------------
# a7: saved-state contract ("activation bytes saved per layer")
# --------------------------------------------------------------------------
def act_saved_bytes(n: int, elem_bytes: int):
    """Exact GELU/SiLU keeps x (n * b bytes); ReGELU2/ReSiLU2 keeps ceil(n/4)
    bytes of codes."""
    return {"exact": int(n) * int(elem_bytes), "ours": codes_bytes(n)}


def norm_saved_bytes(rows: int, cols: int, x_bytes: int):
    """Exact LN/RMSNorm keeps its input x (rows*cols*x_bytes) plus its per-row
    statistics (mean and rstd for LN; the paper counts the input, P:L816,
    P:L824).  MS-LN/MS-RMSNorm keep y, which the next linear layer already
    saves (Prop. 5.1 cond. 3), plus one fp32 rstd per row
    ("one vector ... and one scalar")."""
    return {"exact": int(rows) * int(cols) * int(x_bytes), "ours": 4 * int(rows)}
