"""Build recipe for the native library (nvcc, sm_100a, in-tree output).

Used by ``__graft_entry__.build()`` and, when the shared object is missing
but nvcc is present, by the loader.  Each ``.cu`` compiles to its own
object under ``build/`` (in parallel, rebuilt only when the source or a
header changed), then the objects link into ``lib/libpb_b200.so``.
"""
import os
import shutil
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB_DIR = os.path.join(HERE, "lib")
OBJ_DIR = os.path.join(HERE, "build")
LIB_PATH = os.path.join(LIB_DIR, "libpb_b200.so")
SOURCES = ["pb_capi.cu", "pb_gemm.cu", "pb_factor.cu", "pb_potrf_small.cu", "pb_potrf_reg.cu", "pb_potrf_chain.cu", "pb_trsm_wide.cu", "pb_exact.cu", "pb_pack.cu", "pb_chain.cu", "pb_getrf.cu"]
HEADERS = ["pb_common.cuh", "pb_gemm.cuh", "pb_tri.cuh", "pb_exact.cuh"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC"]


def nvcc_path():
    p = shutil.which("nvcc")
    if p:
        return p
    cand = "/usr/local/cuda/bin/nvcc"
    return cand if os.path.exists(cand) else None


def _headers():
    files = [os.path.join(CSRC, h) for h in HEADERS]
    files.append(os.path.join(os.path.dirname(HERE), "include", "pb_b200.h"))
    return files


def _obj(src):
    return os.path.join(OBJ_DIR, os.path.splitext(src)[0] + ".o")


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(f) > t for f in deps if os.path.exists(f))


def up_to_date():
    if not os.path.exists(LIB_PATH):
        return False
    deps = _headers() + [os.path.join(CSRC, s) for s in SOURCES]
    return not _stale(LIB_PATH, deps)


def build(force=False, verbose=False):
    if not force and up_to_date():
        return LIB_PATH
    nvcc = nvcc_path()
    if nvcc is None:
        raise RuntimeError("nvcc not found: cannot build libpb_b200.so")
    os.makedirs(LIB_DIR, exist_ok=True)
    os.makedirs(OBJ_DIR, exist_ok=True)
    hdrs = _headers()

    def compile_one(src):
        obj = _obj(src)
        path = os.path.join(CSRC, src)
        if not force and not _stale(obj, [path] + hdrs):
            return ""
        tmp = obj + ".tmp%d" % os.getpid()
        res = subprocess.run([nvcc, *NVCC_FLAGS, "-c", "-o", tmp, path], capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError("nvcc failed on %s:\n%s%s" % (src, res.stdout, res.stderr))
        os.replace(tmp, obj)
        return res.stdout + res.stderr

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        logs = list(ex.map(compile_one, SOURCES))
    tmp = LIB_PATH + ".tmp%d" % os.getpid()
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
           "-o", tmp] + [_obj(s) for s in SOURCES]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + res.stdout + res.stderr)
    if verbose:
        print("".join(logs) + res.stdout + res.stderr)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH
