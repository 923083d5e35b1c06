"""C-ABI library checks that need no GPU: the library loads, exports every
symbol include/lmbp.h declares, its host-only entry points behave, and
argument validation returns the documented status codes before any device
work (no compute calls here)."""
import ctypes
import json
import os
import re
from fractions import Fraction

import numpy as np
import pytest

from paper_2406_16282_b200 import _lib, ops

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lmbp.h")
PAPER = json.load(open(os.path.join(ROOT, "tests", "golden", "paper_constants.json")))


def declared_symbols():
    src = open(HEADER).read()
    return re.findall(r"LMBP_API\s+[\w\s\*]+?\b(\w+)\s*\(", src)


def test_header_declares_the_north_star_entry_points():
    names = set(declared_symbols())
    for n in ("regelu2_fwd", "regelu2_bwd", "resilu2_fwd", "resilu2_bwd", "msln_fwd", "msln_bwd", "msrms_fwd", "reswiglu2_fwd", "reswiglu2_bwd",
              "msrms_bwd", "lmbp_codes_bytes", "lmbp_status_string", "lmbp_step_table", "lmbp_version"):
        assert n in names


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    for name in declared_symbols():
        assert hasattr(L, name), name
    assert set(declared_symbols()) == set(_lib.SIGNATURES)
    assert L.lmbp_version().decode().startswith("lmbp")


def test_codes_bytes():
    L = _lib.lib()
    for n in (0, 1, 3, 4, 5, 8, 1_210_368, 452_984_832, -5):
        assert L.lmbp_codes_bytes(n) == (max(n, 0) + 3) // 4


@pytest.mark.parametrize("kind", ["gelu", "silu"])
def test_step_table_is_exact_rounding_of_paper_constants(kind):
    """thresholds = RD32(c) (reading R2): t < c < next_up(t); levels = RN32(s)."""
    thr, lv = ops.step_table(kind)
    for t, cs in zip(thr, PAPER[kind]["c"]):
        c = Fraction(cs)
        t32 = np.float32(t)
        up = np.nextafter(t32, np.float32(np.inf), dtype=np.float32)
        assert Fraction(float(t32)) < c < Fraction(float(up))
    a1, a2 = (float(v) for v in PAPER[kind]["a"])
    want = np.array([0.0, a1, a1 + a2, 1.0]).astype(np.float32)
    assert np.array_equal(np.array(lv, dtype=np.float32), want)


def test_status_strings():
    for st in range(9):
        assert _lib.status_string(st).startswith("LMBP")
    assert "unknown" in _lib.status_string(99)


def test_validation_without_device_work():
    L = _lib.lib()
    S = _lib
    fake = ctypes.c_void_p(0x1000)   # never dereferenced: validation fails first
    for fn in (L.regelu2_fwd, L.resilu2_fwd):
        assert fn(fake, fake, fake, -1, 4, 0, None) == S.LMBP_ERR_SHAPE
        assert fn(fake, fake, fake, 2, 0, 0, None) == S.LMBP_ERR_SHAPE
        assert fn(fake, fake, fake, 2**40, 2**40, 0, None) == S.LMBP_ERR_SHAPE   # int64 overflow
        assert fn(fake, fake, fake, 2, 4, 7, None) == S.LMBP_ERR_DTYPE
        assert fn(None, fake, fake, 2, 4, 0, None) == S.LMBP_ERR_NULLPTR
        assert fn(fake, fake, None, 2, 4, 1, None) == S.LMBP_ERR_NULLPTR
        assert fn(None, None, None, 0, 4, 0, None) == S.LMBP_OK                   # rows == 0: no-op
    for fn in (L.regelu2_bwd, L.resilu2_bwd):
        assert fn(fake, fake, fake, -1, 4, 0, None) == S.LMBP_ERR_SHAPE
        assert fn(fake, None, fake, 2, 4, 2, None) == S.LMBP_ERR_NULLPTR
        assert fn(fake, fake, fake, 2, 4, -1, None) == S.LMBP_ERR_DTYPE
    for fn in (L.msln_fwd, L.msrms_fwd):
        assert fn(fake, fake, fake, 2, 4, 0.0, 0, None) == S.LMBP_ERR_EPS
        assert fn(fake, fake, fake, 2, 4, -1e-6, 0, None) == S.LMBP_ERR_EPS
        assert fn(fake, fake, fake, 2, 4, float("nan"), 0, None) == S.LMBP_ERR_EPS
        assert fn(fake, fake, fake, 2, 4, float("inf"), 0, None) == S.LMBP_ERR_EPS
        assert fn(fake, fake, None, 2, 4, 1e-6, 0, None) == S.LMBP_ERR_NULLPTR
        assert fn(fake, fake, fake, 2, -4, 1e-6, 0, None) == S.LMBP_ERR_SHAPE
        assert fn(fake, fake, fake, 2, 4, 1e-6, 3, None) == S.LMBP_ERR_DTYPE
        assert fn(None, None, None, 0, 4, 1e-6, 0, None) == S.LMBP_OK
    for fn in (L.msln_bwd, L.msrms_bwd):
        assert fn(fake, fake, None, fake, 2, 4, 0, None) == S.LMBP_ERR_NULLPTR
        assert fn(fake, fake, fake, fake, -2, 4, 0, None) == S.LMBP_ERR_SHAPE
        assert fn(fake, fake, fake, fake, 2, 4, 9, None) == S.LMBP_ERR_DTYPE
    assert L.reswiglu2_fwd(fake, fake, fake, fake, fake, -1, 4, 0, None) == S.LMBP_ERR_SHAPE
    assert L.reswiglu2_fwd(fake, None, fake, fake, fake, 2, 4, 0, None) == S.LMBP_ERR_NULLPTR
    assert L.reswiglu2_fwd(fake, fake, fake, fake, fake, 2, 4, 5, None) == S.LMBP_ERR_DTYPE
    assert L.reswiglu2_bwd(fake, fake, fake, None, fake, fake, 2, 4, 1, None) == S.LMBP_ERR_NULLPTR
    assert L.reswiglu2_bwd(fake, fake, fake, fake, fake, fake, 2, 0, 1, None) == S.LMBP_ERR_SHAPE
    assert L.reswiglu2_bwd(None, None, None, None, None, None, 0, 4, 1, None) == S.LMBP_OK
    good = (ctypes.c_double * 3)(-1.0, 0.0, 1.0)
    bad = (ctypes.c_double * 3)(1.0, 0.0, 2.0)
    lv = (ctypes.c_double * 4)(0.0, 0.1, 0.9, 1.0)
    assert L.stepact_fwd(0, 5, ctypes.addressof(good), fake, fake, fake, 2, 4, 0, None) == S.LMBP_ERR_TABLE
    assert L.stepact_fwd(0, 2, ctypes.addressof(bad), fake, fake, fake, 2, 4, 0, None) == S.LMBP_ERR_TABLE
    assert L.stepact_fwd(9, 2, ctypes.addressof(good), fake, fake, fake, 2, 4, 0, None) == S.LMBP_ERR_KIND
    assert L.stepact_fwd(0, 2, None, fake, fake, fake, 2, 4, 0, None) == S.LMBP_ERR_NULLPTR
    assert L.stepact_fwd(0, 2, ctypes.addressof(good), None, fake, fake, 2, 4, 0, None) == S.LMBP_ERR_NULLPTR
    assert L.stepact_bwd(2, ctypes.addressof(lv), fake, fake, fake, -1, 4, 0, None) == S.LMBP_ERR_SHAPE
    assert L.stepact_bwd(5, ctypes.addressof(lv), fake, fake, fake, 2, 4, 0, None) == S.LMBP_ERR_TABLE
    assert L.stepact_bwd(2, ctypes.addressof(lv), None, None, None, 0, 4, 0, None) == S.LMBP_OK
    for k, n in ((1, 9), (2, 9), (4, 9), (3, 9), (5, 9), (2, 0)):
        assert L.lmbp_codes_bytes_k(n, k) == ((n * k + 7) // 8 if k in (1, 2, 3, 4) else 0)
    t = (ctypes.c_float * 4)()
    assert L.lmbp_step_table(5, ctypes.addressof(t), ctypes.addressof(t)) == S.LMBP_ERR_KIND
    assert L.lmbp_step_table(0, None, ctypes.addressof(t)) == S.LMBP_ERR_NULLPTR


def test_binding_refuses_cpu_tensors():
    import torch
    with pytest.raises(ValueError, match="CUDA"):
        ops.regelu2_fwd(torch.zeros(4))
    with pytest.raises(ValueError, match="CUDA"):
        ops.msrms_fwd(torch.zeros(2, 4))


def test_binding_refuses_mixed_devices():
    """Every call runs on one device (the C ABI launches on the current one)."""
    import torch
    a, b = torch.zeros(4), torch.zeros(4, device="meta")
    assert ops._device("f", a, a) == a.device
    with pytest.raises(ValueError, match="different devices"):
        ops._device("f", a, b)


def test_product_package_does_not_import_oracle():
    """The product path never touches oracle/ (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2406_16282_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", src, re.M), f
                assert not re.search(r"#\s*include\s*[<\"].*oracle", src), f
                assert "liboracle" not in src, f


def test_fit_bounds_and_validation_without_device_work():
    """Coefficient fitter (NEXT #4): host-only bounds equal the paper's
    formulas as the oracle implements them; validation precedes device work."""
    from oracle import fit as ofit
    L = _lib.lib()
    S = _lib
    for act in ("gelu", "silu"):
        for eps in (1e-8, 1e-6, 0.5):
            A, B = ops.fit_bounds(act, eps)
            Ao, Bo = ofit.tail_bounds(act, eps)
            assert A == pytest.approx(Ao, rel=1e-15) and B == pytest.approx(Bo, rel=1e-15)
    fake = ctypes.c_void_p(0x1000)
    assert L.lmbp_fit_bounds(7, 1e-8, fake, fake) == S.LMBP_ERR_KIND
    assert L.lmbp_fit_bounds(0, 0.0, ctypes.byref(ctypes.c_double()), ctypes.byref(ctypes.c_double())) == S.LMBP_ERR_EPS
    assert L.lmbp_fit_objective(5, 0, 2, 1e-8, fake, fake, 1, None) == S.LMBP_ERR_KIND
    assert L.lmbp_fit_objective(0, 2, 2, 1e-8, fake, fake, 1, None) == S.LMBP_ERR_KIND
    assert L.lmbp_fit_objective(0, 0, 0, 1e-8, fake, fake, 1, None) == S.LMBP_ERR_SHAPE
    assert L.lmbp_fit_objective(0, 0, 5, 1e-8, fake, fake, 1, None) == S.LMBP_ERR_SHAPE
    assert L.lmbp_fit_objective(0, 0, 2, float("nan"), fake, fake, 1, None) == S.LMBP_ERR_EPS
    assert L.lmbp_fit_objective(0, 0, 2, 1.0, fake, fake, 1, None) == S.LMBP_ERR_EPS
    assert L.lmbp_fit_objective(0, 0, 2, 1e-8, fake, fake, -1, None) == S.LMBP_ERR_SHAPE
    assert L.lmbp_fit_objective(0, 0, 2, 1e-8, None, fake, 1, None) == S.LMBP_ERR_NULLPTR
    assert L.lmbp_fit_objective(0, 0, 2, 1e-8, None, None, 0, None) == S.LMBP_OK
    args = dict(t0=1e-3, t1=1e-9, s0=0.3, s1=1e-6)
    def ann(chains=4, iters=10, t0=1e-3, t1=1e-9, s0=0.3, s1=1e-6, ptr=fake):
        return L.lmbp_fit_anneal(0, 0, 2, 1e-8, None, chains, iters, 1, t0, t1, s0, s1, ptr, ptr, ptr, None)
    assert ann(chains=0) == S.LMBP_ERR_ARG
    assert ann(iters=-1) == S.LMBP_ERR_ARG
    for bad in (0.0, -1.0, float("inf"), float("nan")):
        for key in args:
            kw = dict(args); kw[key] = bad
            assert ann(**kw) == S.LMBP_ERR_ARG
    assert ann(ptr=None) == S.LMBP_ERR_NULLPTR


def test_header_is_plain_c_and_links(tmp_path):
    """The boundary is a C ABI: include/lmbp.h compiles as strict C11, a C
    program links against liblmbp.so and gets the documented host-side
    results (no device work: sizes, status strings, fitter bounds and a
    validation error)."""
    import subprocess
    src = tmp_path / "abi_probe.c"
    src.write_text(r'''
#include <math.h>
#include <stdio.h>
#include <string.h>
#include "lmbp.h"
int main(void) {
  double A = 0.0, B = 0.0;
  float thr[3], lvl[4];
  if (lmbp_codes_bytes(5) != 2 || lmbp_codes_bytes_k(5, 4) != 3) return 1;
  if (strncmp(lmbp_version(), "lmbp", 4) != 0) return 2;
  if (lmbp_fit_bounds(LMBP_GELU, 1e-8, &A, &B) != LMBP_OK || fabs(B - sqrt(-2.0 * log(1e-8))) > 1e-12 || A != -B)
    return 3;
  if (lmbp_step_table(LMBP_SILU, thr, lvl) != LMBP_OK || lvl[3] != 1.0f) return 4;
  if (regelu2_fwd(NULL, NULL, NULL, 4, 8, 9, NULL) != LMBP_ERR_DTYPE) return 5;
  if (msln_fwd(NULL, NULL, NULL, 4, 8, -1.0f, LMBP_F32, NULL) != LMBP_ERR_EPS) return 6;
  printf("%s\n", lmbp_status_string(LMBP_ERR_SHAPE));
  return 0;
}
''')
    lib_dir = os.path.dirname(_lib.LIB)
    exe = tmp_path / "abi_probe"
    subprocess.run(["gcc", "-std=c11", "-pedantic", "-Wall", "-Wextra", "-Werror", f"-I{os.path.join(ROOT, 'include')}",
                    str(src), "-o", str(exe), f"-L{lib_dir}", "-llmbp", f"-Wl,-rpath,{lib_dir}", "-lm"], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, (r.returncode, r.stderr)
    assert r.stdout.startswith("LMBP_ERR_SHAPE")


def test_stepact_binding_refuses_wrong_table_lengths():
    """The C ABI reads exactly 2^k - 1 thresholds / 2^k levels from the host
    pointer: the binding must refuse any other length before the call
    (ADVICE r1), and non-uint8 codes."""
    import torch
    from paper_2406_16282_b200 import ops
    x = torch.zeros(4, 8)
    with pytest.raises(ValueError, match="exactly 15"):
        ops.stepact_fwd(x, "gelu", 4, [-1.0, 0.0, 1.0])         # the 3 published thresholds with k = 4
    with pytest.raises(ValueError, match="exactly 3"):
        ops.stepact_fwd(x, "gelu", 2, [-1.0, 0.0, 1.0, 2.0])
    with pytest.raises(ValueError, match="exactly 8"):
        ops.stepact_bwd(x, torch.zeros(12, dtype=torch.uint8), 3, [0.0] * 7)
    with pytest.raises(ValueError, match="k must be"):
        ops.stepact_fwd(x, "gelu", 5, [0.0] * 31)


def test_mixed_norm_validation_without_device_work():
    """msln/msrms *_mixed: fp32 residual stream with 16-bit y / dy; an fp32 or
    unknown `dtype` is refused, eps and pointers validated as msln_*."""
    L = _lib.lib()
    S = _lib
    fake = ctypes.c_void_p(0x1000)
    for fn in (L.msln_fwd_mixed, L.msrms_fwd_mixed):
        assert fn(fake, fake, fake, 2, 8, 1e-6, S.LMBP_F32, None) == S.LMBP_ERR_DTYPE
        assert fn(fake, fake, fake, 2, 8, 1e-6, 7, None) == S.LMBP_ERR_DTYPE
        assert fn(fake, fake, fake, 2, 8, 0.0, S.LMBP_BF16, None) == S.LMBP_ERR_EPS
        assert fn(fake, None, fake, 2, 8, 1e-6, S.LMBP_F16, None) == S.LMBP_ERR_NULLPTR
        assert fn(fake, fake, fake, -1, 8, 1e-6, S.LMBP_BF16, None) == S.LMBP_ERR_SHAPE
        assert fn(None, None, None, 0, 8, 1e-6, S.LMBP_BF16, None) == S.LMBP_OK
    for fn in (L.msln_bwd_mixed, L.msrms_bwd_mixed):
        assert fn(fake, fake, fake, fake, 2, 8, S.LMBP_F32, None) == S.LMBP_ERR_DTYPE
        assert fn(fake, fake, None, fake, 2, 8, S.LMBP_BF16, None) == S.LMBP_ERR_NULLPTR
        assert fn(None, None, None, None, 0, 8, S.LMBP_F16, None) == S.LMBP_OK


def test_library_provenance_matches_sources():
    """build() records the sha256 of every source the library is compiled
    from next to it (liblmbp.build.json, reported by bench.py); the library in
    the tree was built from the sources in the tree."""
    from paper_2406_16282_b200 import build as B
    info = B.build_info()
    assert info["recorded"] and info["arch"] == "sm_100a"
    assert info["matches_sources"], "liblmbp.so is stale: rebuild with python -m paper_2406_16282_b200.build"
