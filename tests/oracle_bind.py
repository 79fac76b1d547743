"""ctypes bindings for the CPU checkers (test infrastructure only).

- ``orc``: oracle/liboracle.so, our C restatement of the reference path.
- ``ref``: oracle/_ref/libmersenne_ref.so, the unmodified reference sources
  compiled with oracle/ref_shim.cpp (None when it was not built).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "liboracle.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libmersenne_ref.so")

u64 = C.c_uint64
u32 = C.c_uint32
i64 = C.c_int64
P = C.c_void_p
U = C.c_uint
I = C.c_int
D = C.c_double


def _ensure_built():
    if not os.path.exists(ORACLE_SO):
        subprocess.check_call(["make", "-C", ORACLE_DIR, "oracle"], stdout=subprocess.DEVNULL)


def _sig(lib, name, res, args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = args
    return f


def ptr(a):
    if a is None:
        return None
    return C.c_void_p(a.ctypes.data)


class Oracle:
    def __init__(self):
        _ensure_built()
        lib = C.CDLL(ORACLE_SO)
        self.lib = lib
        _sig(lib, "orc_splitmix_next", u64, [P])
        _sig(lib, "orc_splitmix_below", u64, [P, u64])
        _sig(lib, "orc_splitmix_at", u64, [u64, u64])
        _sig(lib, "orc_draw_coeffs", None, [U, U, u64, P, P])
        _sig(lib, "orc_row_seeds", None, [u64, U, P])
        _sig(lib, "orc_hash", I, [U, P, P, U, U, u64, u64, I, P, P])
        _sig(lib, "orc_hash_batch", u64, [U, P, P, U, U, P, u64, P, P])
        _sig(lib, "orc_hash_full_batch", None, [U, P, U, P, u64, P])
        _sig(lib, "orc_mersenne_divmod", I, [U, u64, u64, P, P, P, P])
        _sig(lib, "orc_mersenne_reduce_partial", None, [U, u64, u64, P, P])
        _sig(lib, "orc_pm_setup", U, [U, u64, U, P])
        _sig(lib, "orc_pm_divmod", I, [U, u64, U, P, u64, u64, P, P, P, P])
        _sig(lib, "orc_pm_div_iters", None, [U, u64, U, u64, u64, P, P])
        _sig(lib, "orc_pm_divmod_batch", u64, [U, u64, U, P, P, u64, P, P])
        _sig(lib, "orc_cch_divmod", None, [U, u64, u64, u64, P, P, P, P])
        _sig(lib, "orc_split_pow2", None, [u64, u64, U, U, P, P])
        _sig(lib, "orc_split_arb_uniform", None, [u64, u64, U, u64, P, P])
        _sig(lib, "orc_split_arb_mersenne", None, [u64, u64, U, u64, P, P])
        _sig(lib, "orc_exact_div_iterations", U, [U, u64, u64])
        _sig(lib, "orc_enum_moment_sums", None, [U, u64, I, P, P, u64, P])
        _sig(lib, "orc_bucket_map", u64, [I, U, u64, U, u64, u64])
        _sig(lib, "orc_bucket_map_batch", None, [I, U, u64, U, u64, P, u64, P])
        _sig(lib, "orc_cs_process", u64,
             [U, u64, U, U, P, P, U, I, P, P, P, P, u64, P])
        _sig(lib, "orc_cs_row_moment", None, [P, u64, P, P, P])
        _sig(lib, "orc_cs_second_moment", None, [P, U, u64, I, P, P, P])
        _sig(lib, "orc_cs_point_query", u64, [U, u64, U, U, P, P, U, I, P, P, u64, P])
        _sig(lib, "orc_cs_merge", None, [P, P, u64])
        _sig(lib, "orc_gen_u32_keys", None, [u64, u64, u64, P])
        _sig(lib, "orc_gen_u64_keys", None, [u64, u64, u64, P])
        _sig(lib, "orc_gen_below_p61", u64, [u64, u64, u64, P])
        _sig(lib, "orc_gen_pm_inputs", u64, [u64, u64, u64, u64, P])
        _sig(lib, "orc_zipf_table", None, [D, u32, D, P, P])
        _sig(lib, "orc_gen_zipf_items", None, [u64, P, u32, D, D, u64, u64, P, P])
        _sig(lib, "orc_feistel32", u32, [u64, u32])

    # ---- convenience wrappers (u128 as python int) -------------------------
    def coeffs(self, b, k, seed):
        lo = np.zeros(k, np.uint64)
        hi = np.zeros(k, np.uint64)
        self.lib.orc_draw_coeffs(b, k, seed, ptr(lo), ptr(hi))
        return [int(l) | (int(h) << 64) for l, h in zip(lo, hi)]

    def row_seeds(self, master, rows):
        out = np.zeros(rows, np.uint64)
        self.lib.orc_row_seeds(master, rows, ptr(out))
        return [int(v) for v in out]

    def hash(self, b, coeffs, x, key_bits=None, finish=0):
        k = len(coeffs)
        lo = np.array([c & (2**64 - 1) for c in coeffs], np.uint64)
        hi = np.array([c >> 64 for c in coeffs], np.uint64)
        ol, oh = u64(), u64()
        kb = key_bits if key_bits is not None else 128
        rc = self.lib.orc_hash(b, ptr(lo), ptr(hi), k, kb, x & (2**64 - 1), x >> 64, finish,
                               C.byref(ol), C.byref(oh))
        if rc == 1:
            raise ValueError("key outside domain")
        if rc == 2:
            raise AssertionError("Horner invariant y < 2p violated")
        return ol.value | (oh.value << 64)

    def hash_batch(self, b, coeffs, keys, key_bits):
        k = len(coeffs)
        lo = np.array([c & (2**64 - 1) for c in coeffs], np.uint64)
        hi = np.array([c >> 64 for c in coeffs], np.uint64)
        keys = np.ascontiguousarray(keys, np.uint64)
        ol = np.zeros(len(keys), np.uint64)
        oh = np.zeros(len(keys), np.uint64)
        rej = self.lib.orc_hash_batch(b, ptr(lo), ptr(hi), k, key_bits, ptr(keys), len(keys),
                                      ptr(ol), ptr(oh))
        return ol, oh, rej

    def hash_full(self, b, coeffs, keys):
        c = np.array(coeffs, np.uint64)
        keys = np.ascontiguousarray(keys, np.uint64)
        out = np.zeros(len(keys), np.uint64)
        self.lib.orc_hash_full_batch(b, ptr(c), len(coeffs), ptr(keys), len(keys), ptr(out))
        return out

    def mersenne_divmod(self, b, v):
        ql, qh, rl, rh = u64(), u64(), u64(), u64()
        rc = self.lib.orc_mersenne_divmod(b, v & (2**64 - 1), v >> 64, C.byref(ql), C.byref(qh),
                                          C.byref(rl), C.byref(rh))
        if rc:
            raise ValueError("input exceeds 2^(2b)")
        return ql.value | (qh.value << 64), rl.value | (rh.value << 64)

    def reduce_partial(self, b, y):
        lo, hi = u64(), u64()
        self.lib.orc_mersenne_reduce_partial(b, y & (2**64 - 1), y >> 64, C.byref(lo), C.byref(hi))
        return lo.value | (hi.value << 64)

    def pm_setup(self, b, c, m_iters=0):
        mx = np.zeros(4, np.uint64)
        m = self.lib.orc_pm_setup(b, c, m_iters, ptr(mx))
        if m == 0:
            raise ValueError("invalid pseudo-Mersenne modulus")
        return m, sum(int(v) << (64 * i) for i, v in enumerate(mx)), mx

    def pm_divmod(self, b, c, v, m_iters=0):
        m, _, mx = self.pm_setup(b, c, m_iters)
        ql, qh, rl, rh = u64(), u64(), u64(), u64()
        rc = self.lib.orc_pm_divmod(b, c, m, ptr(mx), v & (2**64 - 1), v >> 64, C.byref(ql),
                                    C.byref(qh), C.byref(rl), C.byref(rh))
        if rc:
            raise ValueError("input exceeds division domain for m iterations")
        return ql.value | (qh.value << 64), rl.value | (rh.value << 64)

    def pm_div_iters(self, b, c, v, iters):
        ql, qh = u64(), u64()
        self.lib.orc_pm_div_iters(b, c, iters, v & (2**64 - 1), v >> 64, C.byref(ql), C.byref(qh))
        return ql.value | (qh.value << 64)

    def pm_divmod_batch(self, b, c, v_lohi, m_iters=0):
        m, _, mx = self.pm_setup(b, c, m_iters)
        v = np.ascontiguousarray(v_lohi, np.uint64)
        n = len(v) // 2
        q = np.zeros(n, np.uint64)
        r = np.zeros(n, np.uint64)
        rej = self.lib.orc_pm_divmod_batch(b, c, m, ptr(mx), ptr(v), n, ptr(q), ptr(r))
        return q, r, rej

    def cch_divmod(self, b, c, v):
        ql, qh, rl, rh = u64(), u64(), u64(), u64()
        self.lib.orc_cch_divmod(b, c, v & (2**64 - 1), v >> 64, C.byref(ql), C.byref(qh),
                                C.byref(rl), C.byref(rh))
        return ql.value | (qh.value << 64), rl.value | (rh.value << 64)

    def split(self, which, h, b, l_or_r):
        idx, sign = u64(), C.c_int()
        fn = [self.lib.orc_split_pow2, self.lib.orc_split_arb_uniform,
              self.lib.orc_split_arb_mersenne][which]
        fn(h & (2**64 - 1), h >> 64, b, l_or_r, C.byref(idx), C.byref(sign))
        return idx.value, sign.value


    def enum_moment_sums(self, b, buckets, splitter, stream):
        keys = np.array([k for k, _ in stream], np.uint64)
        deltas = np.array([d for _, d in stream], np.int64)
        out = np.zeros(4, np.uint64)
        self.lib.orc_enum_moment_sums(b, buckets, splitter, ptr(keys), ptr(deltas), len(keys), ptr(out))
        return int(out[0]) | (int(out[1]) << 64), int(out[2]) | (int(out[3]) << 64)

    def bucket_map(self, kind, b, r, v, c=0):
        """kind 0 map_pow2, 1 map_mersenne, 2 ExactDivisionMap; returns (m, out)."""
        v = np.ascontiguousarray(v, np.uint64)
        m = self.lib.orc_exact_div_iterations(b, c, r) if kind == 2 else 1
        out = np.zeros(len(v), np.uint64)
        if m:
            self.lib.orc_bucket_map_batch(kind, b, c, m, r, ptr(v), len(v), ptr(out))
        return m, out
    def cs_process(self, rows, width, b, coeff_rows, key_bits, splitter, keys, weights=None,
                   counters=None):
        """coeff_rows: list (families) of coefficient lists."""
        k = len(coeff_rows[0])
        flat = [c for row in coeff_rows for c in row]
        lo = np.array([c & (2**64 - 1) for c in flat], np.uint64)
        hi = np.array([c >> 64 for c in flat], np.uint64)
        if counters is None:
            counters = np.zeros(rows * width, np.int64)
        k64 = k32 = w32 = w64 = None
        if keys.dtype == np.uint32:
            k32 = np.ascontiguousarray(keys)
        else:
            k64 = np.ascontiguousarray(keys, np.uint64)
        if weights is not None:
            if weights.dtype == np.int32:
                w32 = np.ascontiguousarray(weights)
            else:
                w64 = np.ascontiguousarray(weights, np.int64)
        rej = self.lib.orc_cs_process(rows, width, b, k, ptr(lo), ptr(hi), key_bits, splitter,
                                      ptr(k64), ptr(k32), ptr(w32), ptr(w64), len(keys),
                                      ptr(counters))
        if rej:
            raise ValueError("key outside domain")
        return counters

    def row_moment(self, counters, width):
        lo, hi, sat = u64(), u64(), C.c_int()
        c = np.ascontiguousarray(counters, np.int64)
        self.lib.orc_cs_row_moment(ptr(c), width, C.byref(lo), C.byref(hi), C.byref(sat))
        return lo.value | (hi.value << 64), bool(sat.value)

    def second_moment(self, counters, rows, width, median=True):
        lo, hi, sat = u64(), u64(), C.c_int()
        c = np.ascontiguousarray(counters, np.int64)
        self.lib.orc_cs_second_moment(ptr(c), rows, width, int(median), C.byref(lo), C.byref(hi),
                                      C.byref(sat))
        return lo.value | (hi.value << 64), bool(sat.value)

    def point_query(self, rows, width, b, coeff_rows, key_bits, splitter, counters, keys):
        k = len(coeff_rows[0])
        flat = [c for row in coeff_rows for c in row]
        lo = np.array([c & (2**64 - 1) for c in flat], np.uint64)
        hi = np.array([c >> 64 for c in flat], np.uint64)
        keys = np.ascontiguousarray(keys, np.uint64)
        out = np.zeros(len(keys), np.int64)
        c = np.ascontiguousarray(counters, np.int64)
        rej = self.lib.orc_cs_point_query(rows, width, b, k, ptr(lo), ptr(hi), key_bits,
                                          splitter, ptr(c), ptr(keys), len(keys), ptr(out))
        if rej:
            raise ValueError("key outside domain")
        return out

    # ---- generators ----------------------------------------------------------
    def gen_u32_keys(self, key_seed, start, n):
        out = np.zeros(n, np.uint32)
        self.lib.orc_gen_u32_keys(key_seed, start, n, ptr(out))
        return out

    def gen_u64_keys(self, key_seed, start, n):
        out = np.zeros(n, np.uint64)
        self.lib.orc_gen_u64_keys(key_seed, start, n, ptr(out))
        return out

    def gen_below_p61(self, key_seed, start, n):
        out = np.zeros(n, np.uint64)
        bad = self.lib.orc_gen_below_p61(key_seed, start, n, ptr(out))
        assert bad == 0
        return out

    def gen_pm_inputs(self, key_seed, c, start, n):
        out = np.zeros(2 * n, np.uint64)
        bad = self.lib.orc_gen_pm_inputs(key_seed, c, start, n, ptr(out))
        assert bad == 0
        return out

    def zipf_table(self, alpha=1.2, T=65536, universe=2.0**32):
        cdf = np.zeros(T, np.uint64)
        c1 = C.c_double()
        self.lib.orc_zipf_table(alpha, T, universe, ptr(cdf), C.byref(c1))
        return cdf, c1.value

    def gen_zipf_items(self, master_seed, start, n, T=65536, universe=2.0**32, table=None):
        cdf, c1 = table if table is not None else self.zipf_table(1.2, T, universe)
        keys = np.zeros(n, np.uint32)
        w = np.zeros(n, np.int32)
        self.lib.orc_gen_zipf_items(master_seed, ptr(cdf), T, c1, universe, start, n, ptr(keys),
                                    ptr(w))
        return keys, w


class Ref:
    """The compiled reference (oracle/_ref)."""

    def __init__(self):
        lib = C.CDLL(REF_SO)
        self.lib = lib
        _sig(lib, "ref_coeffs", I, [U, U, U, u64, P, P])
        _sig(lib, "ref_row_seeds", I, [U, u64, P])
        _sig(lib, "ref_hash_batch", u64, [U, P, P, U, U, I, P, u64, P, P, I])
        _sig(lib, "ref_hash_full_batch", None, [U, P, U, P, u64, P, I])
        _sig(lib, "ref_mersenne_divmod", I, [U, u64, u64, P, P, P, P])
        _sig(lib, "ref_cs_resume", u64, [P, u64, P, P, u64, P, u64, P, P])
        _sig(lib, "ref_two_for_one_run", None, [P, P, U, P, u64, P, I])
        _sig(lib, "ref_pm_setup", U, [U, u64, u64, U, I, P])
        _sig(lib, "ref_pm_divmod_batch", u64, [U, u64, U, P, u64, P, P, I])
        _sig(lib, "ref_pm_divmod", I, [U, u64, U, u64, u64, P, P, P, P])
        _sig(lib, "ref_cch_divmod", None, [U, u64, u64, u64, P, P, P, P])
        _sig(lib, "ref_split", None, [I, u64, u64, U, u64, P, P])
        _sig(lib, "ref_bucket_map", U, [I, U, u64, u64, P, u64, P])
        _sig(lib, "ref_cs_run", I, [U, u64, U, U, I, u64, P, P, P, P, u64, I, P, P])
        _sig(lib, "ref_cs_run_families", I, [U, u64, U, U, I, U, P, P, P, P, u64, P, P])
        _sig(lib, "ref_cs_point_query", I, [U, u64, U, U, I, u64, P, P, u64, P, u64, P])
        _sig(lib, "ref_cs_serialize", u64, [U, u64, U, U, I, u64, P, P, u64, P, u64])
        _sig(lib, "ref_bench_hash", D, [U, U, u64, u64, P])
        _sig(lib, "ref_bench_div", D, [U, u64, u64, u64, P, P])
        _sig(lib, "ref_max_threads", I, [])

    def coeffs(self, b, k, seed, key_bits=32):
        lo = np.zeros(k, np.uint64)
        hi = np.zeros(k, np.uint64)
        assert self.lib.ref_coeffs(b, k, key_bits, seed, ptr(lo), ptr(hi)) == 0
        return [int(l) | (int(h) << 64) for l, h in zip(lo, hi)]

    def row_seeds(self, rows, seed):
        out = np.zeros(rows, np.uint64)
        self.lib.ref_row_seeds(rows, seed, ptr(out))
        return [int(v) for v in out]

    def hash_batch(self, b, coeffs, keys, key_bits, finish=0, threads=1):
        k = len(coeffs)
        lo = np.array([c & (2**64 - 1) for c in coeffs], np.uint64)
        hi = np.array([c >> 64 for c in coeffs], np.uint64)
        keys = np.ascontiguousarray(keys, np.uint64)
        ol = np.zeros(len(keys), np.uint64)
        oh = np.zeros(len(keys), np.uint64)
        rej = self.lib.ref_hash_batch(b, ptr(lo), ptr(hi), k, key_bits, finish, ptr(keys),
                                      len(keys), ptr(ol), ptr(oh), threads)
        return ol, oh, rej

    def hash_full(self, b, coeffs, keys, threads=1):
        c = np.array(coeffs, np.uint64)
        keys = np.ascontiguousarray(keys, np.uint64)
        out = np.zeros(len(keys), np.uint64)
        self.lib.ref_hash_full_batch(b, ptr(c), len(coeffs), ptr(keys), len(keys), ptr(out),
                                     threads)
        return out

    def mersenne_divmod(self, b, v):
        ql, qh, rl, rh = u64(), u64(), u64(), u64()
        rc = self.lib.ref_mersenne_divmod(b, v & (2**64 - 1), v >> 64, C.byref(ql), C.byref(qh),
                                          C.byref(rl), C.byref(rh))
        if rc:
            raise ValueError("input exceeds 2^(2b)")
        return ql.value | (qh.value << 64), rl.value | (rh.value << 64)

    def pm_setup(self, b, c, m_iters=0, engine=0):
        mx = np.zeros(4, np.uint64)
        m = self.lib.ref_pm_setup(b, c & (2**64 - 1), c >> 64, m_iters, engine, ptr(mx))
        if m == 0:
            raise ValueError("invalid pseudo-Mersenne modulus")
        return m, sum(int(v) << (64 * i) for i, v in enumerate(mx))

    def pm_divmod(self, b, c, v, m_iters=0):
        ql, qh, rl, rh = u64(), u64(), u64(), u64()
        rc = self.lib.ref_pm_divmod(b, c, m_iters, v & (2**64 - 1), v >> 64, C.byref(ql),
                                    C.byref(qh), C.byref(rl), C.byref(rh))
        if rc:
            raise ValueError("input exceeds division domain for m iterations")
        return ql.value | (qh.value << 64), rl.value | (rh.value << 64)

    def pm_divmod_batch(self, b, c, v_lohi, m_iters=0, threads=1):
        v = np.ascontiguousarray(v_lohi, np.uint64)
        n = len(v) // 2
        q = np.zeros(n, np.uint64)
        r = np.zeros(n, np.uint64)
        rej = self.lib.ref_pm_divmod_batch(b, c, m_iters, ptr(v), n, ptr(q), ptr(r), threads)
        return q, r, rej

    def cch_divmod(self, b, c, v):
        ql, qh, rl, rh = u64(), u64(), u64(), u64()
        self.lib.ref_cch_divmod(b, c, v & (2**64 - 1), v >> 64, C.byref(ql), C.byref(qh),
                                C.byref(rl), C.byref(rh))
        return ql.value | (qh.value << 64), rl.value | (rh.value << 64)

    def split(self, which, h, b, l_or_r):
        idx, sign = u64(), C.c_int()
        self.lib.ref_split(which, h & (2**64 - 1), h >> 64, b, l_or_r, C.byref(idx),
                           C.byref(sign))
        return idx.value, sign.value


    def bucket_map(self, kind, b, r, v, c=0):
        v = np.ascontiguousarray(v, np.uint64)
        out = np.zeros(len(v), np.uint64)
        m = self.lib.ref_bucket_map(kind, b, c, r, ptr(v), len(v), ptr(out))
        return m, out
    def cs_run(self, rows, width, b, key_bits, splitter, seed, keys, weights=None, threads=1):
        k64 = k32 = w32 = w64 = None
        if keys.dtype == np.uint32:
            k32 = np.ascontiguousarray(keys)
        else:
            k64 = np.ascontiguousarray(keys, np.uint64)
        if weights is not None:
            if weights.dtype == np.int32:
                w32 = np.ascontiguousarray(weights)
            else:
                w64 = np.ascontiguousarray(weights, np.int64)
        counters = np.zeros(rows * width, np.int64)
        mom = np.zeros(3 * (rows + 1), np.uint64)
        rc = self.lib.ref_cs_run(rows, width, b, key_bits, splitter, seed, ptr(k64), ptr(k32),
                                 ptr(w32), ptr(w64), len(keys), threads, ptr(counters), ptr(mom))
        if rc:
            raise ValueError("key outside domain")
        moments = [(int(mom[3 * r]) | (int(mom[3 * r + 1]) << 64), bool(mom[3 * r + 2]))
                   for r in range(rows + 1)]
        return counters, moments[:rows], moments[rows]

    def cs_run_families(self, width, b, key_bits, splitter, coeff_rows, keys, weights=None):
        rows = len(coeff_rows)
        k = len(coeff_rows[0])
        flat = [c for row in coeff_rows for c in row]
        lo = np.array([c & (2**64 - 1) for c in flat], np.uint64)
        hi = np.array([c >> 64 for c in flat], np.uint64)
        keys = np.ascontiguousarray(keys, np.uint64)
        w = None if weights is None else np.ascontiguousarray(weights, np.int64)
        counters = np.zeros(rows * width, np.int64)
        mom = np.zeros(3 * (rows + 1), np.uint64)
        rc = self.lib.ref_cs_run_families(rows, width, b, key_bits, splitter, k, ptr(lo), ptr(hi),
                                          ptr(keys), ptr(w), len(keys), ptr(counters), ptr(mom))
        if rc:
            raise ValueError("key outside domain")
        moments = [(int(mom[3 * r]) | (int(mom[3 * r + 1]) << 64), bool(mom[3 * r + 2]))
                   for r in range(rows + 1)]
        return counters, moments[:rows], moments[rows]

    def point_query(self, rows, width, b, key_bits, splitter, seed, keys, weights, qkeys):
        keys = np.ascontiguousarray(keys, np.uint64)
        w = None if weights is None else np.ascontiguousarray(weights, np.int64)
        q = np.ascontiguousarray(qkeys, np.uint64)
        out = np.zeros(len(q), np.int64)
        rc = self.lib.ref_cs_point_query(rows, width, b, key_bits, splitter, seed, ptr(keys),
                                         ptr(w), len(keys), ptr(q), len(q), ptr(out))
        if rc:
            raise ValueError("key outside domain")
        return out

    def serialize(self, rows, width, b, key_bits, splitter, seed, keys, weights):
        keys = np.ascontiguousarray(keys, np.uint64)
        w = None if weights is None else np.ascontiguousarray(weights, np.int64)
        cap = 64 + 8 * rows + 8 * rows * width
        out = np.zeros(cap, np.uint8)
        n = self.lib.ref_cs_serialize(rows, width, b, key_bits, splitter, seed, ptr(keys), ptr(w),
                                      len(keys), ptr(out), cap)
        return bytes(out[:n])

    def resume(self, payload, keys=None, weights=None):
        """CountSketch::deserialize(payload), process(keys, weights), serialize -> (bytes, median F2)."""
        buf = np.frombuffer(payload, np.uint8).copy()
        keys = np.zeros(0, np.uint64) if keys is None else np.ascontiguousarray(keys, np.uint64)
        w = None if weights is None else np.ascontiguousarray(weights, np.int64)
        out = np.zeros(len(buf) + 64, np.uint8)
        lo, hi = u64(), u64()
        n = self.lib.ref_cs_resume(ptr(buf), len(buf), ptr(keys), ptr(w), len(keys), ptr(out), len(out),
                                   C.byref(lo), C.byref(hi))
        if n == 0:
            raise ValueError("malformed sketch payload")
        return bytes(out[:n]), lo.value | (hi.value << 64)

    def two_for_one(self, coeffs89, keys, threads=1):
        """Config 4's 2 x 65536 table from the reference's hash + split_pow2."""
        lo = np.array([c & (2**64 - 1) for c in coeffs89], np.uint64)
        hi = np.array([c >> 64 for c in coeffs89], np.uint64)
        keys = np.ascontiguousarray(keys, np.uint64)
        table = np.zeros(2 * 65536, np.int64)
        self.lib.ref_two_for_one_run(ptr(lo), ptr(hi), len(coeffs89), ptr(keys), len(keys), ptr(table), threads)
        return table

    def bench_hash(self, b, k, n, seed):
        cs = u64()
        ops = self.lib.ref_bench_hash(b, k, n, seed, C.byref(cs))
        return ops, cs.value

    def bench_div(self, b, c, n, seed):
        cs = u64()
        casc = C.c_double()
        ops = self.lib.ref_bench_div(b, c, n, seed, C.byref(casc), C.byref(cs))
        return ops, casc.value, cs.value


_orc = None
_ref = None


def oracle() -> Oracle:
    global _orc
    if _orc is None:
        _orc = Oracle()
    return _orc


def reference():
    """The compiled reference, or None when oracle/_ref was never built."""
    global _ref
    if _ref is None and os.path.exists(REF_SO):
        _ref = Ref()
    return _ref
