"""Build liblmbp.so (the C-ABI library, include/lmbp.h) in-tree with nvcc for
sm_100a.  No JIT cache: the .so lives next to this file so it travels with the
repository snapshot to the GPU box.

    python -m paper_2406_16282_b200.build [--force]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_obj")
LIB = os.path.join(HERE, "liblmbp.so")
LIB_INFO = os.path.join(HERE, "liblmbp.build.json")   # provenance of LIB (travels with it; not committed)
SOURCES = ["abi.cu", "act.cu", "norm.cu", "norm_mixed.cu", "swiglu.cu", "stepact.cu", "fit.cu"]
HEADERS = ["common.cuh", "constants.cuh", "kernels.h", "act_math.cuh", "act_lut.cuh", "ew_pipeline.cuh",
           os.path.join("..", "..", "include", "lmbp.h"), os.path.join("..", "_obj", "act_lut.inc")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "-Xptxas", "-v", f"-I{os.path.join(ROOT, 'include')}", f"-I{os.path.join(HERE, '_obj')}"]
LUT_INC = os.path.join(HERE, "_obj", "act_lut.inc")


def ensure_lut() -> None:
    """Generate the 16-bit forward tables (lut.py) into _obj/act_lut.inc when
    missing or older than lut.py (build-time constants; not committed)."""
    gen = os.path.join(HERE, "lut.py")
    if _stale(LUT_INC, [gen]):
        os.makedirs(os.path.dirname(LUT_INC), exist_ok=True)
        subprocess.check_call([sys.executable, gen, LUT_INC])


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, objdir: str = OBJ, defines=()) -> str:
    obj = os.path.join(objdir, src.replace(".cu", ".o"))
    deps = [os.path.join(CSRC, src)] + [os.path.join(CSRC, h) for h in HEADERS]
    stamp = obj.replace(".o", ".defines")
    want = "\n".join(sorted(defines))
    try:
        have = open(stamp).read()
    except OSError:
        have = None
    if _stale(obj, deps) or have != want:     # a changed -D set is stale too
        if os.path.exists(stamp):
            os.remove(stamp)
        cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        with open(obj.replace(".o", ".ptxas.log"), "w") as f:
            f.write(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-4000:]}")
        with open(stamp, "w") as f:
            f.write(want)
    return obj


def build(force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    if force:
        for f in os.listdir(OBJ):
            os.remove(os.path.join(OBJ, f))
    ensure_lut()
    with cf.ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(_compile, SOURCES))
    if force or _stale(LIB, objs):
        # cudart is linked statically (nvcc default): one self-contained .so.
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB + ".tmp", *objs]
        subprocess.check_call(cmd)
        os.replace(LIB + ".tmp", LIB)
    if force or _stale(LIB_INFO, [LIB]) or not build_info().get("matches_sources"):
        write_build_info()   # (objects are rebuilt from exactly these sources above)
    return LIB


def source_digest() -> str:
    """sha256 over every file the library is compiled from (kernel sources,
    headers, the C ABI header, the table generator), in a fixed order."""
    import hashlib
    h = hashlib.sha256()
    files = [os.path.join(CSRC, f) for f in SOURCES + HEADERS[:-2]] + \
        [os.path.join(ROOT, "include", "lmbp.h"), os.path.join(HERE, "lut.py")]
    for path in files:
        h.update(os.path.relpath(path, ROOT).encode())
        with open(path, "rb") as f:
            h.update(f.read())
    return h.hexdigest()


def write_build_info() -> None:
    import json
    import time
    try:
        sha = subprocess.run(["git", "-C", ROOT, "rev-parse", "HEAD"], capture_output=True, text=True).stdout.strip()
        dirty = bool(subprocess.run(["git", "-C", ROOT, "status", "--porcelain", "--", "paper_2406_16282_b200/csrc",
                                     "include"], capture_output=True, text=True).stdout.strip())
    except OSError:
        sha, dirty = "", None
    nv = subprocess.run([NVCC, "--version"], capture_output=True, text=True).stdout.strip().splitlines()
    info = {"source_sha256": source_digest(), "git_head": sha or None, "sources_dirty": dirty,
            "nvcc": nv[-1] if nv else None, "arch": "sm_100a",
            "built_utc": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    with open(LIB_INFO, "w") as f:
        json.dump(info, f, indent=1)


def build_info() -> dict:
    """LIB's recorded provenance plus whether it matches the sources present
    now (the check a benchmark or test run reports)."""
    import json
    try:
        info = json.load(open(LIB_INFO))
    except (OSError, ValueError):
        return {"recorded": False}
    info["recorded"] = True
    info["matches_sources"] = info.get("source_sha256") == source_digest()
    return info


def build_variant(name: str, defines, sources=None) -> str:
    """Tuning aid: build liblmbp_<name>.so with extra -D defines into
    _variants/ (used by tools/sweep.py; the product library is LIB)."""
    import hashlib
    tag = hashlib.sha1("\n".join(sorted(defines)).encode()).hexdigest()[:8]
    name = f"{name}-{tag}"                     # same name, different -D set: a different build
    vdir = os.path.join(HERE, "_variant_obj", name)
    os.makedirs(vdir, exist_ok=True)
    ensure_lut()
    srcs = SOURCES if sources is None else list(sources)
    with cf.ThreadPoolExecutor(len(srcs)) as ex:
        objs = list(ex.map(lambda s: _compile(s, vdir, defines), srcs))
    # sources left out are linked from the product build (knob-independent, e.g. fit.cu)
    objs += [_compile(s) for s in SOURCES if s not in srcs]
    os.makedirs(os.path.join(HERE, "_variants"), exist_ok=True)
    out = os.path.join(HERE, "_variants", f"liblmbp_{name}.so")
    if _stale(out, objs) or not os.path.exists(out):
        subprocess.check_call([NVCC, *ARCH, "-shared", "-o", out, *objs])
    import shutil
    shutil.rmtree(vdir, ignore_errors=True)          # objects are only a cache; keep the snapshot small
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
