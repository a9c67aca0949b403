"""ctypes binding of libsvgear.so (C ABI in include/svgear.h).

The shared library is built in-tree from csrc/*.cu by `build_library()` (nvcc, sm_100a only) and
loaded by `lib()`.  There is no fallback of any kind: if the library is missing or a call fails,
an exception is raised.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG_DIR, "csrc")
LIB_PATH = os.path.join(PKG_DIR, "libsvgear.so")
SOURCES = ("api.cu", "kmeans.cu", "lloyd_step.cu", "kmeans_tc.cu", "seed.cu", "seed_ref.cu", "stats_route.cu", "errtab_tc.cu", "attend_ref.cu", "attend_tc.cu", "dit.cu")
NVCC_FLAGS = (
    "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
    "-shared", "-Xcompiler", "-fPIC",
)

OK, EINVAL, ESHAPE, ECUDA, EWORKSPACE, EUNSUPPORTED = 0, -1, -2, -3, -4, -5
EST_VALUE_AWARE, EST_PLAIN = 0, 1
FILL_REMAINDER, STOP_AT_FIRST_OVERFLOW = 0, 1
EXEC_BF16_TENSOR, EXEC_FP32_CHECK = 0, 1
KMEANS_FULL_EVAL = 0x100
ATTEND_ONE_THREAD_PER_ROW, ATTEND_TILE128 = 0x200, 0x400
NORM_NONE, NORM_HEAD, NORM_TOKEN = 0, 1, 2
ROPE_NONE, ROPE_INTERLEAVED, ROPE_HALF_SPLIT = 0, 1, 2


class SvgEarError(RuntimeError):
    """A libsvgear entry point returned a negative status."""

    def __init__(self, fn, status, text):
        super().__init__(f"{fn} failed: {text} (status {status})")
        self.status = status


class Shape(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("bh", "n_q", "n_k", "d", "c_q", "c_k")]


class Aux(C.Structure):
    FIELDS = ("q_assign", "k_assign", "q_perm", "k_perm", "q_sizes", "k_sizes", "q_offsets",
              "k_offsets", "q_centroids", "k_centroids", "v_centroids", "q_iters", "k_iters",
              "error_table", "stabilizers", "mask_entries", "lse")
    _fields_ = [(n, C.c_void_p) for n in FIELDS] + [("kmeans_done_event", C.c_void_p)]


# symbol -> argtypes; every symbol include/svgear.h declares must appear here
_P, _I32, _I64, _SZ = C.c_void_p, C.c_int32, C.c_int64, C.c_size_t
SIGNATURES = {
    "svgear_strerror": ([C.c_int], C.c_char_p),
    "svgear_version": ([], C.c_int),
    "svgear_launch_count": ([], C.c_int64),
    "svgear_workspace_bytes": ([C.POINTER(Shape), C.POINTER(_SZ)], C.c_int),
    "svgear_kmeans": ([_I32, _I32, _I32, _I32, _I32, _P, _P, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P], C.c_int),
    "svgear_kmeans_seed": ([_I32, _I32, _I32, _I32, _P, _I32, C.c_uint32, _I32, _P, _P, _SZ, _P], C.c_int),
    "svgear_kmeans_seed_reference": ([_I32, _I32, _I32, _I32, _P, _P, _P, _P, _P, _SZ, _P], C.c_int),
    "svgear_kmeans_seed_reference_workspace": ([_I32, _I32, C.POINTER(_SZ)], C.c_int),
    "svgear_permute_rows": ([_I32, _I32, _I32, _P, _P, _P, _P], C.c_int),
    "svgear_segment_means": ([_I32, _I32, _I32, _I32, _P, _P, _P, _P, _P], C.c_int),
    "svgear_error_table": ([C.POINTER(Shape), _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P], C.c_int),
    "svgear_route_error_aware": ([_I32, _I32, _I32, _P, _P, _P, _I64, _I32, _I32, _P, _P, _P, _SZ, _P], C.c_int),
    "svgear_route_score": ([C.POINTER(Shape), _P, _P, _P, _P, _I64, _I32, _P, _P, _P, _SZ, _P], C.c_int),
    "svgear_route_score_top_p": ([C.POINTER(Shape), _P, _P, _P, _P, C.c_double, _P, _P, _P, _SZ, _P], C.c_int),
    "svgear_route_error_aware_top_p": ([C.POINTER(Shape), _P, _P, _P, _P, _P, C.c_double, _I32, _I32, _P, _P, _P, _SZ, _P], C.c_int),
    "svgear_sparse_attend": ([C.POINTER(Shape), _I32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P], C.c_int),
    "svgear_forward_seeded": ([C.POINTER(Shape), _P, _P, _P, _I32, C.c_uint32, _I32, _P, _P, _I32, _I32, _I64, _I32, _I32, _I32, C.c_double, _P, _P, C.POINTER(Aux), _P, _SZ, _P], C.c_int),
    "svgear_qkv_prologue": ([_I32, _I32, _I32, _I32, _P, _I32, _P, _P, C.c_float, _I32, _I32, _P, _P, _P, _P, _P, _P], C.c_int),
    "svgear_heads_to_tokens": ([_I32, _I32, _I32, _I32, _P, _P, _P], C.c_int),
    "svgear_forward": ([C.POINTER(Shape), _P, _P, _P, _P, _P, _I32, _I32, _I64, _I32, _I32, _I32, C.c_double, _P, _P, C.POINTER(Aux), _P, _SZ, _P], C.c_int),
}

_lock = threading.Lock()
_lib = None


def _stale():
    if not os.path.exists(LIB_PATH):
        return True
    t = os.path.getmtime(LIB_PATH)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [
        os.path.join(os.path.dirname(PKG_DIR), "include", "svgear.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def build_library(force=False, verbose=False):
    """Compile csrc/*.cu into libsvgear.so for sm_100a (nvcc cross-compiles without a GPU).  Each
    source becomes an object under build/ (recompiled only when it or a header changed, in
    parallel), then one link step."""
    if not force and not _stale():
        return LIB_PATH
    from concurrent.futures import ThreadPoolExecutor

    obj_dir = os.path.join(PKG_DIR, "build")
    os.makedirs(obj_dir, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))] + [
        os.path.join(os.path.dirname(PKG_DIR), "include", "svgear.h")]
    newest_header = max(os.path.getmtime(h) for h in headers)
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"]

    def compile_one(src):
        path = os.path.join(CSRC, src)
        obj = os.path.join(obj_dir, src[:-3] + ".o")
        if not force and os.path.exists(obj) and os.path.getmtime(obj) > max(os.path.getmtime(path), newest_header):
            return obj, ""
        cmd = ["nvcc", *compile_flags, "-c", "-o", obj, path]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n" + res.stdout + res.stderr)
        return obj, res.stderr

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as pool:
        results = list(pool.map(compile_one, SOURCES))
    if verbose:
        print("".join(err for _, err in results))
    link = ["nvcc", "-shared", "-Xcompiler", "-fPIC", "-gencode", "arch=compute_100a,code=sm_100a", "-o", LIB_PATH,
            *[obj for obj, _ in results], "-lcuda"]
    res = subprocess.run(link, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + res.stdout + res.stderr)
    return LIB_PATH


def lib():
    """Load libsvgear.so (building it first only if nvcc is available and it is missing)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                build_library()
            handle = C.CDLL(LIB_PATH)
            for name, (args, res) in SIGNATURES.items():
                fn = getattr(handle, name)  # AttributeError if the symbol is not exported
                fn.argtypes = args
                fn.restype = res
            _lib = handle
        return _lib


def check(fn_name, status):
    if status != OK:
        raise SvgEarError(fn_name, status, lib().svgear_strerror(status).decode())


def workspace_bytes(shape: Shape) -> int:
    out = _SZ(0)
    check("svgear_workspace_bytes", lib().svgear_workspace_bytes(C.byref(shape), C.byref(out)))
    return int(out.value)
