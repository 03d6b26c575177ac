"""Build + load the C oracle (TEST INFRASTRUCTURE ONLY)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
BUILD = os.path.join(HERE, "_build")
NUMERICS_SO = os.path.join(BUILD, "libnumerics_ref.so")
REF_DIR = os.path.join(HERE, "_ref")


def build_numerics() -> str:
    src = os.path.join(HERE, "numerics_ref.c")
    if not os.path.exists(NUMERICS_SO) or os.path.getmtime(NUMERICS_SO) < os.path.getmtime(src):
        os.makedirs(BUILD, exist_ok=True)
        subprocess.check_call(["gcc", "-O3", "-march=x86-64-v3", "-shared", "-fPIC", "-pthread", src,
                               "-o", NUMERICS_SO, "-lm"])
    return NUMERICS_SO


def build_reference() -> bool:
    """Compile the reference in place into oracle/_ref (needs /root/reference)."""
    if not os.path.isdir("/root/reference/proj"):
        return os.path.exists(os.path.join(REF_DIR, "muxsim"))
    subprocess.check_call(["make", "-s", "-j8", "-C", HERE])
    return True


_lib = None


def numerics() -> C.CDLL:
    global _lib
    if _lib is None:
        lib = C.CDLL(build_numerics())
        P = C.c_void_p
        lib.ref_decode_attention.argtypes = [P, P, P, P, P, P, C.c_int, C.c_int, C.c_int, C.c_int,
                                             C.c_int, P, C.c_int]
        lib.ref_gemv_bf16.argtypes = [P, P, P, C.c_int, C.c_int, C.c_int, C.c_int]
        lib.ref_f32_to_bf16.argtypes = [P, P, C.c_int64]
        _lib = lib
    return _lib


def decode_attention(q_u16, pool_u16, rowrec, rowlist, slots, ctx, L, layer, max_rows, nthreads=8):
    """numpy in/out wrapper around ref_decode_attention (fp32 [B][H][128])."""
    import numpy as np
    B, H = q_u16.shape[0], q_u16.shape[1]
    out = np.zeros((B, H, 128), np.float32)
    arrs = [np.ascontiguousarray(a) for a in (q_u16, pool_u16, rowrec, rowlist, slots, ctx)]
    numerics().ref_decode_attention(*[a.ctypes.data for a in arrs], B, H, L, layer, max_rows,
                                    out.ctypes.data, nthreads)
    return out
