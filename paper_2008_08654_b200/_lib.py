"""ctypes binding of the C-ABI boundary (include/mersenne_b200.h).

The product path has no CPU fallback: importing this module without the built
library raises ImportError, and every device entry fails with CudaError when
no sm_100 GPU is visible.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmersenne_b200.so")
HARNESS_PATH = os.path.join(HERE, "libmersenne_b200_harness.so")

MB200_OK = 0
MB200_INVALID_ARGUMENT = 1
MB200_DOMAIN_ERROR = 2
MB200_LOGIC_ERROR = 3
MB200_CUDA_ERROR = 4
MB200_UNSUPPORTED = 5

KEY_U32, KEY_U64 = 32, 64
W_NONE, W_I32, W_I64 = 0, 32, 64
SPLIT_POW2, SPLIT_UNIFORM_ARB, SPLIT_MERSENNE_ARB, SPLIT_TWO_FOR_ONE = 0, 1, 2, 3
MAP_POW2, MAP_MERSENNE, MAP_EXACT_DIV = 0, 1, 2


class InvalidArgument(ValueError):
    """std::invalid_argument of the reference (construction-time checks)."""


class DomainError(ValueError):
    """std::domain_error of the reference (key / dividend outside the domain)."""


class LogicError(RuntimeError):
    """std::logic_error of the reference."""


class CudaError(RuntimeError):
    """CUDA failure, or no usable sm_100 device (there is no CPU fallback)."""


class Unsupported(NotImplementedError):
    """Valid for the reference but not implemented on the GPU path."""


_EXC = {
    MB200_INVALID_ARGUMENT: InvalidArgument,
    MB200_DOMAIN_ERROR: DomainError,
    MB200_LOGIC_ERROR: LogicError,
    MB200_CUDA_ERROR: CudaError,
    MB200_UNSUPPORTED: Unsupported,
}

u64, u32, i64, i32 = C.c_uint64, C.c_uint32, C.c_int64, C.c_int32
P, U, I, D = C.c_void_p, C.c_uint, C.c_int, C.c_double


class SketchDesc(C.Structure):
    _fields_ = [
        ("rows", U),
        ("width", u64),
        ("b", U),
        ("k", U),
        ("key_bits", U),
        ("splitter", I),
        ("coeffs_lo", P),
        ("coeffs_hi", P),
    ]


# (name, restype, argtypes) of every exported entry in include/mersenne_b200.h
SIGNATURES = [
    ("mb200_last_error", C.c_char_p, []),
    ("mb200_abi_version", I, []),
    ("mb200_device_count", I, []),
    ("mb200_mersenne_modulus_check", I, [U, I]),
    ("mb200_pm_modulus", I, [U, u64, u64, U, P, P]),
    ("mb200_draw_coeffs", I, [U, U, u64, P, P]),
    ("mb200_precondition61", I, [P, P]),
    ("mb200_row_seeds", I, [u64, U, P]),
    ("mb200_hash61", I, [P, I, u64, U, P, U, U, P, P]),
    ("mb200_hash89", I, [P, u64, P, P, U, U, P, P, P]),
    ("mb200_hash_wide", I, [P, u64, U, P, P, U, U, P, P, P]),
    ("mb200_pm_divmod", I, [P, u64, U, u64, U, P, P, P, P]),
    ("mb200_pm_div", I, [P, u64, U, u64, U, P, P, P]),
    ("mb200_pm_mod", I, [P, P, u64, U, u64, P, P]),
    ("mb200_mersenne_divmod", I, [P, u64, U, P, P, P]),
    ("mb200_split_batch", I, [I, P, u64, U, u64, P, P, P, P]),
    ("mb200_exact_division_iterations", I, [U, u64, u64, P]),
    ("mb200_bucket_map", I, [I, P, u64, U, u64, u64, P, P, P]),
    ("mb200_enum_moment_sums", I, [U, u64, u64, I, P, P, u64, P, P]),
    ("mb200_cs_update", I, [P, P, I, P, I, u64, P, P]),
    ("mb200_cs_moments", I, [P, U, u64, P, P]),
    ("mb200_cs_merge", I, [P, P, u64, P]),
    ("mb200_cs_point_query", I, [P, P, P, I, u64, P, P]),
    ("mb200_sketch_create", I, [U, u64, U, U, I, u64, U, P]),
    ("mb200_sketch_create_families", I, [u64, I, U, U, U, U, P, P, U, P]),
    ("mb200_sketch_destroy", None, [P]),
    ("mb200_sketch_process", I, [P, P, I, P, I, u64]),
    ("mb200_sketch_process_device", I, [P, P, I, P, I, u64, P]),
    ("mb200_sketch_h2d_bytes", I, [P, P]),
    ("mb200_set_host_threads", None, [I]),
    ("mb200_host_threads", I, []),
    ("mb200_sketch_row_second_moment", I, [P, U, P, P, P]),
    ("mb200_sketch_second_moment", I, [P, I, P, P, P]),
    ("mb200_sketch_point_query", I, [P, P, I, u64, P]),
    ("mb200_sketch_merge", I, [P, P]),
    ("mb200_sketch_counters", I, [P, P]),
    ("mb200_sketch_set_counters", I, [P, P]),
    ("mb200_sketch_device_counters", P, [P]),
    ("mb200_sketch_info", I, [P, P, P, P, P, P, P]),
    ("mb200_sketch_seeds", I, [P, P]),
    ("mb200_sketch_coeffs", I, [P, P, P]),
    ("mb200_sketch_serialize", I, [P, P, u64, P]),
    ("mb200_sketch_deserialize", I, [P, u64, P]),
    ("mb200_nccl_version", I, [P]),
    ("mb200_nccl_unique_id", I, [P]),
    ("mb200_nccl_comm_init", I, [I, P, I, P]),
    ("mb200_nccl_comm_destroy", I, [P]),
    ("mb200_nccl_comm_size", I, [P, P]),
    ("mb200_cs_allreduce", I, [P, u64, P, P]),
    ("mb200_sketch_allreduce", I, [P, P]),
    ("mb200_hot_stats", I, [P, I]),
    ("mb200_kernel_timer", I, [I]),
    ("mb200_kernel_timer_read", I, [P, P]),
    ("mb200_set_large_table_strategy", I, [I, P]),
]


# bench / test harness library (include/mersenne_b200_harness.h): not the drop-in ABI
HARNESS_SIGNATURES = [
    ("mb200_gen_u32_keys", I, [u64, u64, u64, P, P]),
    ("mb200_gen_u64_keys", I, [u64, u64, u64, P, P]),
    ("mb200_gen_below_p61", I, [u64, u64, u64, P, P, P]),
    ("mb200_gen_pm_inputs", I, [u64, u64, u64, u64, P, P, P]),
    ("mb200_zipf_table", I, [D, u32, D, P, P]),
    ("mb200_gen_zipf_items", I, [u64, P, u32, D, D, u64, u64, P, P, P]),
    ("mb200_probe_imad", I, [I, I, I, P, P]),
    ("mb200_probe_atomics", I, [I, I, I, I, P, u64, P]),
    ("mb200_probe_dsmem", I, [I, I, I, I, I, u32, P, P]),
]


def _bind(lib, sigs):
    for name, res, args in sigs:
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


def _preload_bundled_nccl():
    """The library binds NCCL at run time (host/nccl_comm.cpp): the one already in the
    process, else the loader's libnccl.so.2.  In a Python process that imports torch LATER,
    a system libnccl loaded first would satisfy torch's own libnccl.so.2 dependency by
    soname -- and an older one lacks symbols torch needs.  So the NCCL wheel torch was
    built against (nvidia/nccl/lib), when installed, is loaded first; without it nothing
    changes."""
    import glob
    import importlib.util

    try:
        spec = importlib.util.find_spec("nvidia.nccl")
        for base in (spec.submodule_search_locations if spec else []) or []:
            for f in sorted(glob.glob(os.path.join(base, "lib", "libnccl.so*"))):
                C.CDLL(f, mode=C.RTLD_GLOBAL)
                return
    except (ImportError, OSError, ValueError):
        pass


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "or `make lib` (the B200 path has no CPU fallback)")
    _preload_bundled_nccl()
    return _bind(C.CDLL(LIB_PATH), SIGNATURES)


lib = _load()
_harness = None


def harness():
    """The bench harness library (generators, probes), loaded on first use."""
    global _harness
    if _harness is None:
        if not os.path.exists(HARNESS_PATH):
            raise ImportError(f"{HARNESS_PATH} is not built: run `make lib`")
        _harness = _bind(C.CDLL(HARNESS_PATH), HARNESS_SIGNATURES)
    return _harness


def check(status: int) -> None:
    if status != MB200_OK:
        msg = lib.mb200_last_error().decode()
        raise _EXC.get(status, RuntimeError)(msg)
