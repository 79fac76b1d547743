"""B200-native Mersenne-prime hashing and Count Sketch (arXiv 2008.08654 hot path).

Python face of the C-ABI in include/mersenne_b200.h.  Names follow the
reference library (/root/reference/proj/include/mersenne/*.hpp): the
``CountSketch`` object mirrors mersenne::CountSketch (sketch.hpp:40-92) on
host buffers, and the device-array functions (``hash61``, ``cs_update``, ...)
take torch CUDA tensors (torch is plumbing: device memory and streams).

All arithmetic runs in hand-written sm_100a kernels; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from ._lib import (  # noqa: F401
    KEY_U32, KEY_U64, LIB_PATH, MAP_EXACT_DIV, MAP_MERSENNE, MAP_POW2, SIGNATURES, SPLIT_MERSENNE_ARB, SPLIT_POW2, SPLIT_TWO_FOR_ONE,
    SPLIT_UNIFORM_ARB, W_I32, W_I64, W_NONE, CudaError, DomainError, InvalidArgument, LogicError,
    SketchDesc, Unsupported, check, harness, lib,
)

MASK64 = (1 << 64) - 1
SALT_KEYS = 0x7B5BAD595E238E31  # bench.cpp:23 key-stream salt


def _p(a: np.ndarray):
    return C.c_void_p(a.ctypes.data) if a is not None else None


def device_count() -> int:
    return lib.mb200_device_count()


# ------------------------------------------------------------------ field / draws
def mersenne_modulus_check(b: int, require_prime: bool = False) -> None:
    check(lib.mb200_mersenne_modulus_check(b, int(require_prime)))


def pm_modulus(b: int, c: int, m_iters: int = 0):
    """PseudoMersenneModulus(b, c, m_iters) -> (iterations, max_input)."""
    m = C.c_uint()
    mx = np.zeros(4, np.uint64)
    check(lib.mb200_pm_modulus(b, c & MASK64, c >> 64, m_iters, C.byref(m), _p(mx)))
    return m.value, sum(int(v) << (64 * i) for i, v in enumerate(mx))


def draw_coeffs(b: int, k: int, seed: int) -> list:
    """PolyHashFamily(MersenneModulus(b), k, u, seed).coefficients() (polyhash.cpp:12-35)."""
    lo = np.zeros(k, np.uint64)
    hi = np.zeros(k, np.uint64)
    check(lib.mb200_draw_coeffs(b, k, seed & MASK64, _p(lo), _p(hi)))
    return [int(l) | (int(h) << 64) for l, h in zip(lo, hi)]


def precondition61(coeffs) -> dict | None:
    """Adapted coefficients of a degree-7 polynomial over Z_(2^61-1) (mb200_precondition61):
    {"al": [al0..al5], "s": shift, "a7": leading coefficient, "r0": remainder}, or None when
    the leading coefficient is 0 (the hash kernel then evaluates by Horner)."""
    c = np.array([int(v) for v in coeffs], np.uint64)
    if c.size != 8:
        raise ValueError("precondition61 takes 8 coefficients")
    plan = np.zeros(9, np.uint64)
    rc = lib.mb200_precondition61(_p(c), _p(plan))
    if rc == 5:  # MB200_UNSUPPORTED: leading coefficient 0
        return None
    check(rc)
    v = [int(x) for x in plan]
    return {"al": v[:6], "s": v[6], "a7": v[7], "r0": v[8]}


def row_seeds(master: int, rows: int) -> list:
    out = np.zeros(rows, np.uint64)
    check(lib.mb200_row_seeds(master & MASK64, rows, _p(out)))
    return [int(v) for v in out]


# ------------------------------------------------------------------ torch plumbing
def _torch():
    import torch

    return torch


def _stream(stream):
    torch = _torch()
    if stream is None:
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


def _key_width(t) -> int:
    torch = _torch()
    if t.dtype in (torch.int32, torch.uint32):
        return 32
    if t.dtype in (torch.int64, torch.uint64):
        return 64
    raise InvalidArgument(f"keys must be a 32- or 64-bit integer tensor, got {t.dtype}")


def _weight_kind(t) -> int:
    torch = _torch()
    if t is None:
        return W_NONE
    if t.dtype == torch.int32:
        return W_I32
    if t.dtype == torch.int64:
        return W_I64
    raise InvalidArgument(f"weights must be int32 or int64, got {t.dtype}")


def _dptr(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise InvalidArgument("device entry needs CUDA tensors")
    if not t.is_contiguous():
        raise InvalidArgument("tensors must be contiguous")
    return C.c_void_p(t.data_ptr())


def hash61(keys, coeffs: Sequence[int], b: int = 61, key_bits: Optional[int] = None, out=None,
           stream=None):
    """Alg 1 mod 2^b - 1 (b <= 61) over a device key tensor; returns int64 tensor of u64 hashes."""
    torch = _torch()
    kw = _key_width(keys)
    n = keys.numel()
    if out is None:
        out = torch.empty(n, dtype=torch.int64, device=keys.device)
    c = np.array([int(a) & MASK64 for a in coeffs], np.uint64)
    kb = kw if key_bits is None else key_bits
    check(lib.mb200_hash61(_dptr(keys), kw, n, b, _p(c), len(coeffs), kb, _dptr(out), _stream(stream)))
    return out


def hash89(keys, coeffs: Sequence[int], key_bits: int = 64, out_lo=None, out_hi=None, stream=None):
    """Alg 1 mod 2^89 - 1 over u64 device keys; returns (low 64 bits, high 25 bits)."""
    torch = _torch()
    n = keys.numel()
    if out_lo is None:
        out_lo = torch.empty(n, dtype=torch.int64, device=keys.device)
    if out_hi is None:
        out_hi = torch.empty(n, dtype=torch.int64, device=keys.device)
    lo = np.array([int(a) & MASK64 for a in coeffs], np.uint64)
    hi = np.array([int(a) >> 64 for a in coeffs], np.uint64)
    check(lib.mb200_hash89(_dptr(keys), n, _p(lo), _p(hi), len(coeffs), key_bits, _dptr(out_lo),
                           _dptr(out_hi), _stream(stream)))
    return out_lo, out_hi


def hash_wide(keys, b: int, coeffs: Sequence[int], key_bits: int = 64, out_lo=None, out_hi=None, stream=None):
    """Alg 1 mod 2^b - 1 for 62 <= b <= 127 (the reference's generic path) over u64
    device keys; returns (low 64 bits, high bits)."""
    torch = _torch()
    n = keys.numel()
    if out_lo is None:
        out_lo = torch.empty(n, dtype=torch.int64, device=keys.device)
    if out_hi is None:
        out_hi = torch.empty(n, dtype=torch.int64, device=keys.device)
    lo = np.array([int(a) & MASK64 for a in coeffs], np.uint64)
    hi = np.array([int(a) >> 64 for a in coeffs], np.uint64)
    check(lib.mb200_hash_wide(_dptr(keys), n, b, _p(lo), _p(hi), len(coeffs), key_bits, _dptr(out_lo),
                              _dptr(out_hi), _stream(stream)))
    return out_lo, out_hi


def pm_divmod(v, b: int, c: int, m_iters: int = 0, q=None, r=None, overflow=None, stream=None):
    """Alg 4 + Alg 5 by p = 2^b - c over u128 inputs stored as an (n, 2) int64 tensor of
    (lo, hi) words; returns (q, r) int64 tensors holding u64 values."""
    torch = _torch()
    n = v.numel() // 2
    if q is None:
        q = torch.empty(n, dtype=torch.int64, device=v.device)
    if r is None:
        r = torch.empty(n, dtype=torch.int64, device=v.device)
    check(lib.mb200_pm_divmod(_dptr(v), n, b, c, m_iters, _dptr(q), _dptr(r), _dptr(overflow),
                              _stream(stream)))
    return q, r


def pm_div(v, b: int, c: int, m_iters: int = 0, q=None, overflow=None, stream=None):
    """pseudo_mersenne_div (field.cpp:260-265) alone: quotients of (n, 2) u128 inputs."""
    torch = _torch()
    n = v.numel() // 2
    if q is None:
        q = torch.empty(n, dtype=torch.int64, device=v.device)
    check(lib.mb200_pm_div(_dptr(v), n, b, c, m_iters, _dptr(q), _dptr(overflow), _stream(stream)))
    return q


def pm_mod(v, z, b: int, c: int, r=None, stream=None):
    """pseudo_mersenne_mod (field.cpp:267-273): (v + z c) & (2^b - 1) for given quotients z."""
    torch = _torch()
    n = v.numel() // 2
    if r is None:
        r = torch.empty(n, dtype=torch.int64, device=v.device)
    check(lib.mb200_pm_mod(_dptr(v), _dptr(z), n, b, c, _dptr(r), _stream(stream)))
    return r


def mersenne_divmod(v, b: int, q=None, r=None, stream=None):
    """mersenne_divmod, Alg 3 (field.cpp:208-222), over (n, 2) u128 inputs < 2^(2b)."""
    torch = _torch()
    n = v.numel() // 2
    if q is None:
        q = torch.empty(n, dtype=torch.int64, device=v.device)
    if r is None:
        r = torch.empty(n, dtype=torch.int64, device=v.device)
    check(lib.mb200_mersenne_divmod(_dptr(v), n, b, _dptr(q), _dptr(r), _stream(stream)))
    return q, r


def split_batch(splitter: int, h, b: int, l_or_r: int, index=None, sign=None, out_of_domain=None,
                stream=None):
    """split_pow2 / split_arb_uniform / split_arb_mersenne (sketch.cpp:13-34) of a device
    batch of u64 hash values; returns (index int64, sign int32 of +1/-1)."""
    torch = _torch()
    n = h.numel()
    if index is None:
        index = torch.empty(n, dtype=torch.int64, device=h.device)
    if sign is None:
        sign = torch.empty(n, dtype=torch.int32, device=h.device)
    check(lib.mb200_split_batch(splitter, _dptr(h), n, b, l_or_r, _dptr(index), _dptr(sign),
                                _dptr(out_of_domain), _stream(stream)))
    return index, sign


def exact_division_iterations(b: int, c: int, r: int) -> int:
    """ExactDivisionMap(PseudoMersenneModulus(b, c), r).divider().iterations()
    (bucketing.cpp:75-89)."""
    m = C.c_uint()
    check(lib.mb200_exact_division_iterations(b, c, r, C.byref(m)))
    return m.value


def bucket_map(kind: int, v, b: int, r: int, c: int = 0, out=None, out_of_domain=None, stream=None):
    """Bucket map of a device u64 batch (int64 tensor): MAP_POW2 map_pow2(v, b, r),
    MAP_MERSENNE map_mersenne(v, b, r), MAP_EXACT_DIV ExactDivisionMap(PseudoMersenneModulus(b, c), r)(v)
    (bucketing.cpp:61-95).  Values outside the domain raise DomainError unless
    `out_of_domain` (device int64[1]) collects their count asynchronously."""
    torch = _torch()
    if out is None:
        out = torch.empty(v.numel(), dtype=torch.int64, device=v.device)
    check(lib.mb200_bucket_map(kind, _dptr(v), v.numel(), b, c, r, _dptr(out), _dptr(out_of_domain),
                               _stream(stream)))
    return out


class ExactDivisionMap:
    """bucketing.hpp:43-58: v -> floor(v r / p) on [0, p), p = 2^b - c, via Alg 4 with the
    iteration count grown until (p-1) r is admissible.  Calls run on the GPU."""

    def __init__(self, b: int, c: int, r: int):
        self.m = exact_division_iterations(b, c, r)
        self.b, self.c, self.r = b, c, r
        self.p = (1 << b) - c

    def buckets(self) -> int:
        return self.r

    def iterations(self) -> int:
        return self.m

    def __call__(self, v, out=None, stream=None):
        return bucket_map(MAP_EXACT_DIV, v, self.b, self.r, self.c, out=out, stream=stream)


def enum_moment_sums(b: int, buckets: int, splitter: int, stream, key_domain: Optional[int] = None,
                     stream_=None) -> dict:
    """enum_moment_sums (verify.cpp:575-603) on the GPU: over all p^4 degree-3 families
    (p = 2^b - 1) of a one-row sketch with `buckets` counters, exact sums of
    X = sum C_i^2 and X^2.  stream: [(key, delta), ...] with distinct keys mod p."""
    keys = np.array([int(k) for k, _ in stream], np.uint64)
    deltas = np.array([int(d) for _, d in stream], np.int64)
    if key_domain is None:
        key_domain = (1 << b) - 1
    out = np.zeros(5, np.uint64)
    check(lib.mb200_enum_moment_sums(b, key_domain, buckets, splitter, _p(keys), _p(deltas), len(keys),
                                     _p(out), _stream(stream_) if stream_ is not None else None))
    return {"sum_x": int(out[0]) | (int(out[1]) << 64), "sum_x_sq": int(out[2]) | (int(out[3]) << 64),
            "families": int(out[4])}


def enum_sketch_moments(b: int, buckets: int, splitter: int, stream, key_domain: Optional[int] = None) -> dict:
    """The three exact checks of enum_sketch_moments (verify.cpp:605-653) from the GPU sums:
    the mean equals (F2 p^2 + F1^2 - F2) / p^2, lies within F2 (n-1)/p^2 of F2, and the
    variance is below 2 F2^2 / r (Pow2) or 2 F2^2 (2^(2b) + r^2) / (r 2^(2b)).  Values are
    exact fractions.  (The reference's JSON report/budget layer is out of scope.)"""
    from fractions import Fraction as Fr

    s = enum_moment_sums(b, buckets, splitter, stream, key_domain)
    p = (1 << b) - 1
    f1 = sum(int(d) for _, d in stream)
    f2 = sum(int(d) * int(d) for _, d in stream)
    fam, p2, n = s["families"], p * p, len(stream)
    mean = Fr(s["sum_x"], fam)
    formula = Fr(f2 * p2 + f1 * f1 - f2, p2)
    tol = Fr(f2 * (n - 1), p2)
    var = Fr(s["sum_x_sq"], fam) - mean * mean
    bound = (Fr(2 * f2 * f2, buckets) if splitter == SPLIT_POW2 else
             Fr(2 * f2 * f2 * ((1 << (2 * b)) + buckets * buckets), buckets << (2 * b)))
    checks = [("mean matches exact formula", mean, formula, "=="),
              ("mean within relative distance of F2", abs(mean - f2), tol, "<="),
              ("variance below bound", var, bound, "<=")]
    return {"sums": s, "checks": [{"name": nm, "value": v, "bound": bd, "relation": rel,
                                   "pass": v == bd if rel == "==" else v <= bd} for nm, v, bd, rel in checks]}


class SketchSpec:
    """Geometry + coefficients of a sketch, as the mb200_sketch_desc the kernels take."""

    def __init__(self, rows: int, width: int, b: int, families: Sequence[Sequence[int]],
                 key_bits: int, splitter: int = SPLIT_POW2):
        self.rows, self.width, self.b, self.key_bits, self.splitter = rows, width, b, key_bits, splitter
        self.families = [list(f) for f in families]
        self.k = len(self.families[0])
        flat = [int(a) for f in self.families for a in f]
        self._lo = np.array([a & MASK64 for a in flat], np.uint64)
        self._hi = np.array([a >> 64 for a in flat], np.uint64)
        self.desc = SketchDesc(rows, width, b, self.k, key_bits, splitter,
                               self._lo.ctypes.data, self._hi.ctypes.data)

    @classmethod
    def seeded(cls, rows, width, b=61, key_bits=32, splitter=SPLIT_POW2, seed=1, independence=4):
        """CountSketch(rows, width, MersenneModulus(b), 2^key_bits, splitter, seed) families."""
        fams = (rows + 1) // 2 if splitter == SPLIT_TWO_FOR_ONE else rows
        seeds = row_seeds(seed, fams)
        return cls(rows, width, b, [draw_coeffs(b, independence, s) for s in seeds], key_bits,
                   splitter)


def set_host_threads(n: int) -> None:
    """Host threads CountSketch.process packs and checks with (0 = automatic)."""
    lib.mb200_set_host_threads(int(n))


def host_threads() -> int:
    return lib.mb200_host_threads()


def cs_update(spec: SketchSpec, keys, counters, weights=None, stream=None):
    """Fused K3+K4 scatter of a device batch into `counters` (int64, rows*width)."""
    check(lib.mb200_cs_update(C.byref(spec.desc), _dptr(keys), _key_width(keys), _dptr(weights),
                              _weight_kind(weights), keys.numel(), _dptr(counters), _stream(stream)))
    return counters


def cs_moments(counters, rows: int, width: int, out=None, stream=None):
    """K5: per-row (value lo, value hi, saturated, 0) as an int64 (rows, 4) tensor."""
    torch = _torch()
    if out is None:
        out = torch.empty((rows, 4), dtype=torch.int64, device=counters.device)
    check(lib.mb200_cs_moments(_dptr(counters), rows, width, _dptr(out), _stream(stream)))
    return out


def moments_to_python(m) -> list:
    """(rows, 4) moment tensor -> [(value, saturated)] with exact ints."""
    a = m.cpu().numpy().astype(np.uint64)
    return [(int(r[0]) | (int(r[1]) << 64), bool(r[2])) for r in a]


def lower_median(moments: list):
    """second_moment(true): lower median of rows by value (sketch.cpp:160-168)."""
    s = sorted(moments, key=lambda t: t[0])
    return s[(len(s) - 1) // 2]


def cs_merge(dst, src, stream=None):
    check(lib.mb200_cs_merge(_dptr(dst), _dptr(src), dst.numel(), _stream(stream)))
    return dst


def cs_point_query(spec: SketchSpec, counters, keys, out=None, stream=None):
    torch = _torch()
    if out is None:
        out = torch.empty(keys.numel(), dtype=torch.int64, device=keys.device)
    check(lib.mb200_cs_point_query(C.byref(spec.desc), _dptr(counters), _dptr(keys), _key_width(keys),
                                   keys.numel(), _dptr(out), _stream(stream)))
    return out


# ------------------------------------------------------------------ multi-GPU merge
def nccl_version() -> int:
    v = C.c_int()
    check(lib.mb200_nccl_version(C.byref(v)))
    return v.value


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    check(lib.mb200_nccl_unique_id(buf))
    return bytes(buf)


class NcclComm:
    """One NCCL communicator over the ranks of a job (one GPU per rank), made by the
    product library (mb200_nccl_comm_init on the current device).  ``cs_allreduce`` /
    ``CountSketch.allreduce`` sum the rank-local tables through it."""

    def __init__(self, nranks: int, uid: bytes, rank: int):
        if len(uid) != 128:
            raise InvalidArgument("NCCL unique id must be 128 bytes")
        h = C.c_void_p()
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        check(lib.mb200_nccl_comm_init(nranks, buf, rank, C.byref(h)))
        self._h, self.nranks, self.rank = h, nranks, rank

    @classmethod
    def from_process_group(cls, group=None) -> "NcclComm":
        """Rank 0 draws the unique id and torch.distributed (any backend) ships it."""
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls(world, obj[0], rank)

    @property
    def ptr(self):
        return self._h

    def size(self) -> int:
        n = C.c_int()
        check(lib.mb200_nccl_comm_size(self._h, C.byref(n)))
        return n.value

    def close(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and lib is not None:
            lib.mb200_nccl_comm_destroy(h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter teardown
            pass


def cs_allreduce(counters, comm: NcclComm, stream=None):
    """In-place NCCL sum of the rank-local tables (distributed CountSketch::merge,
    sketch.cpp:182-193); asynchronous on `stream`."""
    check(lib.mb200_cs_allreduce(_dptr(counters), counters.numel(), comm.ptr, _stream(stream)))
    return counters


# ------------------------------------------------------------------ generators
def gen_u32_keys(seed: int, start: int, n: int, out=None, stream=None):
    torch = _torch()
    out = torch.empty(n, dtype=torch.int32, device="cuda") if out is None else out
    check(harness().mb200_gen_u32_keys(seed & MASK64, start, n, _dptr(out), _stream(stream)))
    return out


def gen_u64_keys(seed: int, start: int, n: int, out=None, stream=None):
    torch = _torch()
    out = torch.empty(n, dtype=torch.int64, device="cuda") if out is None else out
    check(harness().mb200_gen_u64_keys(seed & MASK64, start, n, _dptr(out), _stream(stream)))
    return out


def gen_below_p61(seed: int, start: int, n: int, out=None, bad=None, stream=None):
    torch = _torch()
    out = torch.empty(n, dtype=torch.int64, device="cuda") if out is None else out
    bad = torch.zeros(1, dtype=torch.int64, device="cuda") if bad is None else bad
    check(harness().mb200_gen_below_p61(seed & MASK64, start, n, _dptr(out), _dptr(bad), _stream(stream)))
    return out, bad


def gen_pm_inputs(seed: int, c: int, start: int, n: int, out=None, bad=None, stream=None):
    torch = _torch()
    out = torch.empty((n, 2), dtype=torch.int64, device="cuda") if out is None else out
    bad = torch.zeros(1, dtype=torch.int64, device="cuda") if bad is None else bad
    check(harness().mb200_gen_pm_inputs(seed & MASK64, c, start, n, _dptr(out), _dptr(bad),
                                  _stream(stream)))
    return out, bad


def zipf_table(alpha: float = 1.2, T: int = 65536, universe: float = 2.0 ** 32):
    cdf = np.zeros(T, np.uint64)
    c1 = C.c_double()
    check(harness().mb200_zipf_table(alpha, T, universe, _p(cdf), C.byref(c1)))
    return cdf, c1.value


class ZipfStream:
    """Config-5 item stream: Zipf(1.2) ranks over 2^32 keys (seeded Feistel rank->key
    permutation) with int32 weights in [-100, 100]; counter-addressable by item index."""

    def __init__(self, master_seed: int = 1, T: int = 65536, universe: float = 2.0 ** 32):
        torch = _torch()
        self.master, self.T, self.universe = master_seed & MASK64, T, universe
        cdf, self.c1 = zipf_table(1.2, T, universe)
        self.cdf_host = cdf
        self.cdf = torch.from_numpy(cdf.view(np.int64)).cuda()

    def generate(self, start: int, n: int, keys=None, weights=None, stream=None):
        torch = _torch()
        keys = torch.empty(n, dtype=torch.int32, device="cuda") if keys is None else keys
        weights = torch.empty(n, dtype=torch.int32, device="cuda") if weights is None else weights
        check(harness().mb200_gen_zipf_items(self.master, _dptr(self.cdf), self.T, self.c1, self.universe,
                                       start, n, _dptr(keys), _dptr(weights), _stream(stream)))
        return keys, weights


def probe_imad(blocks: int, threads: int, iters: int, sink, stream=None):
    check(harness().mb200_probe_imad(blocks, threads, iters, _dptr(sink), _stream(stream)))


def probe_atomics(mode: int, blocks: int, threads: int, iters: int, buf, span: int, stream=None):
    check(harness().mb200_probe_atomics(mode, blocks, threads, iters, _dptr(buf), span, _stream(stream)))


def probe_dsmem(cluster: int, mode: int, blocks: int, threads: int, iters: int, words: int, out,
                stream=None):
    check(harness().mb200_probe_dsmem(cluster, mode, blocks, threads, iters, words, _dptr(out), _stream(stream)))


def kernel_timer(enable: bool = True) -> None:
    """Bench hook: CUDA events around the dominant scatter kernel of every
    large-table cs_update (mb200_kernel_timer)."""
    check(lib.mb200_kernel_timer(int(enable)))


def kernel_timer_read():
    """(summed kernel seconds, launches) since the timer was enabled / last read."""
    ms = C.c_double()
    n = C.c_uint64()
    check(lib.mb200_kernel_timer_read(C.byref(ms), C.byref(n)))
    return ms.value / 1e3, n.value


def hot_stats(reset: bool = False) -> dict:
    """Counters of the heavy-hitter Count Sketch kernel since the last reset."""
    out = np.zeros(8, np.uint64)
    check(lib.mb200_hot_stats(_p(out), int(reset)))
    return {"items": int(out[0]), "misses": int(out[1]), "hot_applied": int(out[2]), "hot_keys": int(out[3]),
            "binned": int(out[4]), "direct": int(out[5]), "bin_merges": int(out[6]), "raw_batches": int(out[7])}


LARGE_DIRECT, LARGE_BINNED, LARGE_ROWS = 0, 1, 2


def set_large_table_strategy(strategy: int) -> int:
    """Route hot-set misses of large tables to L2 reductions (LARGE_DIRECT, default) or
    through HBM bins (LARGE_BINNED) or through the miss buffer and per-row passes
    (LARGE_ROWS); returns the previous strategy."""
    prev = C.c_int(0)
    check(lib.mb200_set_large_table_strategy(int(strategy), C.byref(prev)))
    return prev.value


# ------------------------------------------------------------------ host object
class CountSketch:
    """mersenne::CountSketch (sketch.hpp:40-92) with counters in HBM; host-buffer API."""

    def __init__(self, rows: int, width: int, b: int = 61, key_bits: int = 32,
                 splitter: int = SPLIT_POW2, seed: int = 1, independence: int = 4, _handle=None):
        if _handle is not None:
            self._h = _handle
        else:
            h = C.c_void_p()
            check(lib.mb200_sketch_create(rows, width, b, key_bits, splitter, seed & MASK64,
                                          independence, C.byref(h)))
            self._h = h
        self._info()

    @classmethod
    def from_families(cls, width: int, splitter: int, b: int, key_bits: int,
                      families: Sequence[Sequence[int]], rows: int = 0):
        """CountSketch(width, splitter, families) (sketch.cpp:84-95)."""
        k = len(families[0])
        flat = [int(a) for f in families for a in f]
        lo = np.array([a & MASK64 for a in flat], np.uint64)
        hi = np.array([a >> 64 for a in flat], np.uint64)
        h = C.c_void_p()
        check(lib.mb200_sketch_create_families(width, splitter, b, key_bits, len(families), k, _p(lo),
                                               _p(hi), rows, C.byref(h)))
        return cls(0, 0, _handle=h)

    def _info(self):
        rows, width, b, k, kb, sp = C.c_uint(), C.c_uint64(), C.c_uint(), C.c_uint(), C.c_uint(), C.c_int()
        check(lib.mb200_sketch_info(self._h, C.byref(rows), C.byref(width), C.byref(b), C.byref(k),
                                    C.byref(kb), C.byref(sp)))
        self.rows, self.width, self.b = rows.value, width.value, b.value
        self.independence, self.key_bits, self.splitter = k.value, kb.value, sp.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and lib is not None:
            try:
                lib.mb200_sketch_destroy(h)
            except Exception:  # interpreter teardown
                pass
            self._h = None

    def process(self, keys, weights=None):
        """process(key, delta) for every item of host arrays (numpy)."""
        keys = np.ascontiguousarray(keys)
        if keys.dtype not in (np.uint32, np.int32, np.uint64, np.int64):
            keys = keys.astype(np.uint64)
        kw = 32 if keys.dtype.itemsize == 4 else 64
        wk = W_NONE
        if weights is not None:
            weights = np.ascontiguousarray(weights)
            if weights.dtype == np.int32:
                wk = W_I32
            else:
                weights = weights.astype(np.int64)
                wk = W_I64
        check(lib.mb200_sketch_process(self._h, _p(keys), kw, _p(weights), wk, len(keys)))

    def h2d_bytes(self) -> int:
        """Bytes process() has moved host -> device (deltas narrowed when they fit)."""
        v = C.c_uint64()
        check(lib.mb200_sketch_h2d_bytes(self._h, C.byref(v)))
        return v.value

    def process_one(self, key: int, delta: int):
        self.process(np.array([key], np.uint64), np.array([delta], np.int64))

    def process_device(self, keys, weights=None, stream=None):
        check(lib.mb200_sketch_process_device(self._h, _dptr(keys), _key_width(keys), _dptr(weights),
                                              _weight_kind(weights), keys.numel(), _stream(stream)))

    def row_second_moment(self, row: int):
        lo, hi, sat = C.c_uint64(), C.c_uint64(), C.c_int()
        check(lib.mb200_sketch_row_second_moment(self._h, row, C.byref(lo), C.byref(hi), C.byref(sat)))
        return lo.value | (hi.value << 64), bool(sat.value)

    def second_moment(self, median_rows: bool = False):
        lo, hi, sat = C.c_uint64(), C.c_uint64(), C.c_int()
        check(lib.mb200_sketch_second_moment(self._h, int(median_rows), C.byref(lo), C.byref(hi),
                                             C.byref(sat)))
        return lo.value | (hi.value << 64), bool(sat.value)

    def point_query(self, keys):
        keys = np.ascontiguousarray(keys)
        kw = 32 if keys.dtype.itemsize == 4 else 64
        if kw == 64:
            keys = keys.astype(np.uint64)
        out = np.zeros(len(keys), np.int64)
        check(lib.mb200_sketch_point_query(self._h, _p(keys), kw, len(keys), _p(out)))
        return out

    def merge(self, other: "CountSketch"):
        check(lib.mb200_sketch_merge(self._h, other._h))
        return self

    def allreduce(self, comm: "NcclComm"):
        """merge() across the ranks of `comm`: the replicas' HBM tables are summed in place."""
        check(lib.mb200_sketch_allreduce(self._h, comm.ptr))
        return self

    def counters(self) -> np.ndarray:
        out = np.zeros(self.rows * self.width, np.int64)
        check(lib.mb200_sketch_counters(self._h, _p(out)))
        return out

    def set_counters(self, c: np.ndarray):
        c = np.ascontiguousarray(c, np.int64)
        check(lib.mb200_sketch_set_counters(self._h, _p(c)))

    def device_counters_ptr(self) -> int:
        return lib.mb200_sketch_device_counters(self._h)

    def seeds(self) -> list:
        fams = (self.rows + 1) // 2 if self.splitter == SPLIT_TWO_FOR_ONE else self.rows
        out = np.zeros(fams, np.uint64)
        check(lib.mb200_sketch_seeds(self._h, _p(out)))
        return [int(v) for v in out]

    def serialize(self) -> bytes:
        """MCSK1 bytes, identical to mersenne::CountSketch::serialize (sketch.cpp:195-211)."""
        n = C.c_uint64()
        check(lib.mb200_sketch_serialize(self._h, None, 0, C.byref(n)))
        buf = np.zeros(n.value, np.uint8)
        check(lib.mb200_sketch_serialize(self._h, _p(buf), n.value, C.byref(n)))
        return buf.tobytes()

    @classmethod
    def deserialize(cls, payload: bytes) -> "CountSketch":
        """mersenne::CountSketch::deserialize (sketch.cpp:213-244)."""
        buf = np.frombuffer(payload, np.uint8).copy()
        h = C.c_void_p()
        check(lib.mb200_sketch_deserialize(_p(buf) if len(buf) else None, len(buf), C.byref(h)))
        return cls(0, 0, _handle=h)

    def coefficients(self) -> list:
        fams = (self.rows + 1) // 2 if self.splitter == SPLIT_TWO_FOR_ONE else self.rows
        lo = np.zeros(fams * self.independence, np.uint64)
        hi = np.zeros(fams * self.independence, np.uint64)
        check(lib.mb200_sketch_coeffs(self._h, _p(lo), _p(hi)))
        flat = [int(l) | (int(h) << 64) for l, h in zip(lo, hi)]
        k = self.independence
        return [flat[i * k:(i + 1) * k] for i in range(fams)]
