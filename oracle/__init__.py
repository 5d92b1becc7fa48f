"""TEST INFRASTRUCTURE ONLY — the checker, never the product.

numpy front-ends for
  * ``liboracle.so``: this repo's plain-C restatement of the reference hot path
    (oracle/oracle.c, each function citing the reference file:line), and
  * ``_ref/libspmvkit_ref.so``: the UNMODIFIED reference library compiled in
    place from /root/reference/proj/core by oracle/Makefile (glue:
    oracle/ref_capi.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(paper_1012_2270_b200, libspmvk.so) never does.

Parity status: PINNED.  The restatement is checked against the reference
itself (tests/test_oracle_pinned.py, when _ref is built) and against the golden
vectors tests/golden/*.npz generated from the reference by
oracle/make_golden.py.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libspmvkit_ref.so")

_O = None
_R = None


def build(quiet: bool = True) -> None:
    """Builds liboracle.so and (when /root/reference exists) _ref/."""
    subprocess.run(["make", "-C", HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _ptr(a):
    return a.ctypes.data if a is not None and a.size else None


def O():
    """liboracle.so (restatement), loaded once."""
    global _O
    if _O is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        u64, vp, ci, dbl = C.c_uint64, C.c_void_p, C.c_int, C.c_double
        sig = {
            "orc_random_vector": (None, [u64, u64, vp]),
            "orc_random_matrix": (u64, [u64, u64, dbl, ci, ci, ci, ci, u64, vp, vp, vp]),
            "orc_random_small_spec": (None, [u64, vp, vp, vp, vp]),
            "orc_banded": (u64, [u64, u64, u64, vp, vp, vp]),
            "orc_spmv_reference": (None, [u64, vp, vp, vp, vp, vp]),
            "orc_spmv_csr_f64": (None, [u64, vp, vp, vp, vp, vp]),
            "orc_spmv_csr_f32": (None, [u64, vp, vp, vp, vp, vp]),
            "orc_rgcsr_layout": (u64, [u64, vp, u64, vp, vp, vp]),
            "orc_rgcsr_fill_f64": (None, [u64, vp, vp, vp, u64, vp, vp, vp]),
            "orc_rgcsr_fill_f32": (None, [u64, vp, vp, vp, u64, vp, vp, vp]),
            "orc_spmv_rgcsr_f64": (u64, [u64, u64, vp, vp, vp, vp, vp, vp]),
            "orc_spmv_rgcsr_f32": (u64, [u64, u64, vp, vp, vp, vp, vp, vp]),
            "orc_hybrid_split_cost": (u64, [vp, u64, u64]),
            "orc_choose_ell_width": (u64, [vp, u64]),
            "orc_hybrid_coo_count": (u64, [u64, vp, u64]),
            "orc_hybrid_fill_f64": (None, [u64, vp, vp, vp, u64, vp, vp, vp, vp, vp]),
            "orc_hybrid_fill_f32": (None, [u64, vp, vp, vp, u64, vp, vp, vp, vp, vp]),
            "orc_spmv_hybrid_f64": (None, [u64, u64, vp, vp, u64, vp, vp, vp, vp, vp]),
            "orc_spmv_hybrid_f32": (None, [u64, u64, vp, vp, u64, vp, vp, vp, vp, vp]),
            "orc_descending_map": (None, [u64, vp, vp]),
            "orc_stencil": (u64, [ci, u64, vp, vp, vp]),
            "orc_powerlaw": (u64, [u64, u64, vp, vp, vp]),
        }
        for k, (r, a) in sig.items():
            f = getattr(L, k)
            f.restype, f.argtypes = r, a
        _O = L
    return _O


class Csr:
    """Canonical matrix as host CSR (== the reference's sorted TripletMatrix)."""

    def __init__(self, rows, cols, rp, col, val):
        self.rows, self.cols = int(rows), int(cols)
        self.rp = np.ascontiguousarray(rp, np.uint32)
        self.col = np.ascontiguousarray(col, np.uint32)
        self.val = np.ascontiguousarray(val, np.float64)

    @property
    def nnz(self):
        return int(self.col.size)

    def lens(self):
        return np.diff(self.rp.astype(np.int64)).astype(np.uint64)


# ------------------------------------------------------------------ generators
def random_vector(n, seed):
    out = np.empty(n, np.float64)
    O().orc_random_vector(n, seed, _ptr(out))
    return out


def random_matrix(rows, cols, density, vmin, vmax, integer, allow_zero, seed):
    L = O()
    rp = np.empty(rows + 1, np.uint32)
    nnz = L.orc_random_matrix(rows, cols, density, vmin, vmax, int(integer), int(allow_zero),
                              seed, None, None, None)
    col = np.empty(nnz, np.uint32)
    val = np.empty(nnz, np.float64)
    L.orc_random_matrix(rows, cols, density, vmin, vmax, int(integer), int(allow_zero), seed,
                        _ptr(rp), _ptr(col), _ptr(val))
    return Csr(rows, cols, rp, col, val)


def random_small(seed, allow_zero=True, integer=True):
    """tests/fixtures.hpp:50-60 random_small."""
    r, c, d, s = C.c_uint64(), C.c_uint64(), C.c_double(), C.c_uint64()
    O().orc_random_small_spec(seed, C.byref(r), C.byref(c), C.byref(d), C.byref(s))
    return random_matrix(r.value, c.value, d.value, -8, 8, integer, allow_zero, s.value)


def random_case(seed, max_rows):
    """tests/acceptance.cpp:87-94 random_case: random_small's draw order with
    the shape drawn modulo max_rows."""
    st = _MT(seed)
    rows = 1 + st.next() % max_rows
    cols = 1 + st.next() % max_rows
    density = 0.05 + 0.25 * st.unit_real()
    mseed = st.next()
    return random_matrix(rows, cols, density, -8, 8, True, True, mseed)


class _MT:
    """std::mt19937_64 in Python (small draws only; mirrors orc_mt64)."""

    def __init__(self, seed):
        self.mt = [0] * 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) \
                & 0xFFFFFFFFFFFFFFFF
        self.i = 312

    def next(self):
        M = 0xFFFFFFFFFFFFFFFF
        if self.i >= 312:
            um, lm = 0xFFFFFFFF80000000, 0x7FFFFFFF
            for k in range(312):
                x = (self.mt[k] & um) | (self.mt[(k + 1) % 312] & lm)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                self.mt[k] = self.mt[(k + 156) % 312] ^ xa
            self.i = 0
        x = self.mt[self.i]
        self.i += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000 & M
        x ^= (x << 37) & 0xFFF7EEE000000000 & M
        x ^= x >> 43
        return x & M

    def unit_real(self):
        return float(self.next() >> 11) * 2.0 ** -53


def random_integer_x(n, seed):
    """tests/acceptance.cpp:96-101: rng() % 17 - 8 per element."""
    st = _MT(seed)
    return np.array([float((st.next() % 17) - 8) for _ in range(n)], np.float64)


def banded(n, hbw, seed):
    L = O()
    nnz = L.orc_banded(n, hbw, seed, None, None, None)
    rp, col, val = np.empty(n + 1, np.uint32), np.empty(nnz, np.uint32), np.empty(nnz)
    L.orc_banded(n, hbw, seed, _ptr(rp), _ptr(col), _ptr(val))
    return Csr(n, n, rp, col, val)


def stencil(kind, n):
    L = O()
    rows = n * n if kind == 5 else n ** 3
    nnz = L.orc_stencil(kind, n, None, None, None)
    rp, col, val = np.empty(rows + 1, np.uint32), np.empty(nnz, np.uint32), np.empty(nnz)
    L.orc_stencil(kind, n, _ptr(rp), _ptr(col), _ptr(val))
    return Csr(rows, rows, rp, col, val)


def powerlaw(rows, seed=7):
    L = O()
    nnz = L.orc_powerlaw(rows, seed, None, None, None)
    rp, col, val = np.empty(rows + 1, np.uint32), np.empty(nnz, np.uint32), np.empty(nnz)
    L.orc_powerlaw(rows, seed, _ptr(rp), _ptr(col), _ptr(val))
    return Csr(rows, rows, rp, col, val)


# ------------------------------------------------------------------ formats
def spmv_reference(m: Csr, x):
    y = np.empty(m.rows, np.float64)
    O().orc_spmv_reference(m.rows, _ptr(m.rp), _ptr(m.col), _ptr(m.val),
                           _ptr(np.ascontiguousarray(x, np.float64)), _ptr(y))
    return y


def spmv_csr(m: Csr, x, prec=8):
    dt = np.float64 if prec == 8 else np.float32
    y = np.empty(m.rows, dt)
    val = m.val.astype(dt)
    fn = O().orc_spmv_csr_f64 if prec == 8 else O().orc_spmv_csr_f32
    fn(m.rows, _ptr(m.rp), _ptr(m.col), _ptr(val), _ptr(np.ascontiguousarray(x, dt)), _ptr(y))
    return y


def build_rgcsr(m: Csr, G, prec=8):
    """build_rgcsr<S> (rgcsr.hpp:38-70) -> dict of the four arrays; raises
    ValueError for G == 0 and OverflowError when slots exceed uint32."""
    if G == 0:
        raise ValueError("build_rgcsr: group size must be nonzero")
    L = O()
    groups = (m.rows + G - 1) // G
    lens = np.empty(m.rows, np.uint32)
    gp = np.empty(groups + 1, np.uint32)
    ovf = C.c_int()
    slots = L.orc_rgcsr_layout(m.rows, _ptr(m.rp), G, _ptr(lens), _ptr(gp), C.byref(ovf))
    if ovf.value:
        raise OverflowError(f"{slots} slots overflow uint32")
    dt = np.float64 if prec == 8 else np.float32
    values = np.empty(slots, dt)
    columns = np.empty(slots, np.uint32)
    fn = L.orc_rgcsr_fill_f64 if prec == 8 else L.orc_rgcsr_fill_f32
    fn(m.rows, _ptr(m.rp), _ptr(m.col), _ptr(m.val), G, _ptr(gp), _ptr(values), _ptr(columns))
    return dict(values=values, columns=columns, group_pointers=gp, row_lengths=lens,
                group_size=G, rows=m.rows, cols=m.cols)


def spmv_rgcsr(a: dict, x):
    dt = a["values"].dtype
    y = np.empty(a["rows"], dt)
    fn = O().orc_spmv_rgcsr_f64 if dt == np.float64 else O().orc_spmv_rgcsr_f32
    madds = fn(a["rows"], a["group_size"], _ptr(a["group_pointers"]), _ptr(a["row_lengths"]),
               _ptr(a["values"]), _ptr(a["columns"]), _ptr(np.ascontiguousarray(x, dt)), _ptr(y))
    return y, madds


def rgcsr_fill(a: dict):
    """(slots, nnz, artificial_zeros, bytes_single, bytes_double) per fill.hpp:90-95."""
    slots = int(a["values"].size)
    nnz = int(a["row_lengths"].astype(np.uint64).sum())
    words = slots + a["group_pointers"].size + a["row_lengths"].size
    return slots, nnz, slots - nnz, slots * 4 + words * 4, slots * 8 + words * 4


def hybrid_split_cost(lens, k):
    L = np.ascontiguousarray(lens, np.uint64)
    return int(O().orc_hybrid_split_cost(_ptr(L), L.size, k))


def choose_ell_width(lens):
    L = np.ascontiguousarray(lens, np.uint64)
    return int(O().orc_choose_ell_width(_ptr(L), L.size))


def build_hybrid(m: Csr, k1=None, prec=8):
    L = O()
    if k1 is None:
        k1 = choose_ell_width(m.lens())
    coo = L.orc_hybrid_coo_count(m.rows, _ptr(m.rp), k1)
    if coo == 2 ** 64 - 1:
        raise ValueError(f"build_hybrid: k1 {k1} exceeds the maximum row length")
    dt = np.float64 if prec == 8 else np.float32
    out = dict(ell_values=np.empty(m.rows * k1, dt), ell_columns=np.empty(m.rows * k1, np.uint32),
               coo_rows=np.empty(coo, np.uint32), coo_columns=np.empty(coo, np.uint32),
               coo_values=np.empty(coo, dt), k1=k1, rows=m.rows, cols=m.cols)
    fn = L.orc_hybrid_fill_f64 if prec == 8 else L.orc_hybrid_fill_f32
    fn(m.rows, _ptr(m.rp), _ptr(m.col), _ptr(m.val), k1, _ptr(out["ell_values"]),
       _ptr(out["ell_columns"]), _ptr(out["coo_rows"]), _ptr(out["coo_columns"]),
       _ptr(out["coo_values"]))
    return out


def spmv_hybrid(h: dict, x):
    dt = h["ell_values"].dtype
    y = np.empty(h["rows"], dt)
    fn = O().orc_spmv_hybrid_f64 if dt == np.float64 else O().orc_spmv_hybrid_f32
    fn(h["rows"], h["k1"], _ptr(h["ell_values"]), _ptr(h["ell_columns"]), h["coo_rows"].size,
       _ptr(h["coo_rows"]), _ptr(h["coo_columns"]), _ptr(h["coo_values"]),
       _ptr(np.ascontiguousarray(x, dt)), _ptr(y))
    return y


def descending_map(m: Csr):
    out = np.empty(m.rows, np.uint32)
    O().orc_descending_map(m.rows, _ptr(m.rp), _ptr(out))
    return out


# ------------------------------------------------------------------ the reference itself
def ref_available() -> bool:
    return os.path.exists(REF_SO)


def R():
    """_ref/libspmvkit_ref.so (the unmodified reference), loaded once."""
    global _R
    if _R is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference)")
        L = C.CDLL(REF_SO)
        u64, vp, ci, dbl, i64 = C.c_uint64, C.c_void_p, C.c_int, C.c_double, C.c_int64
        pp = C.POINTER(C.c_void_p)
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_tm_from_csr": (ci, [u64, u64, u64, vp, vp, vp, pp]),
            "ref_tm_example8": (ci, [pp]),
            "ref_tm_random_small": (ci, [u64, ci, ci, pp]),
            "ref_tm_random_case": (ci, [u64, u64, pp]),
            "ref_tm_random_matrix": (ci, [u64, u64, dbl, ci, ci, ci, ci, u64, pp]),
            "ref_tm_banded": (ci, [u64, u64, u64, pp]),
            "ref_tm_descending": (ci, [vp, pp]),
            "ref_descending_map": (ci, [vp, vp]),
            "ref_tm_dims": (None, [vp, vp, vp, vp]),
            "ref_tm_export": (None, [vp, vp, vp, vp]),
            "ref_tm_free": (None, [vp]),
            "ref_spmv_reference": (ci, [vp, vp, u64, vp]),
            "ref_random_vector": (None, [u64, u64, vp]),
            "ref_measured_gflops": (dbl, [u64, dbl]),
            "ref_csr_build": (ci, [vp, ci, pp]),
            "ref_csr_spmv": (ci, [vp, vp, u64, vp, u64]),
            "ref_csr_free": (None, [vp]),
            "ref_rgcsr_build": (ci, [vp, u64, ci, pp]),
            "ref_rgcsr_info": (None, [vp, vp]),
            "ref_rgcsr_export": (None, [vp, vp, vp, vp, vp]),
            "ref_rgcsr_spmv": (ci, [vp, vp, u64, vp, u64, vp]),
            "ref_rgcsr_free": (None, [vp]),
            "ref_choose_ell_width": (u64, [vp, u64]),
            "ref_hybrid_split_cost": (u64, [vp, u64, u64]),
            "ref_hybrid_build": (ci, [vp, i64, ci, pp]),
            "ref_hybrid_info": (None, [vp, vp]),
            "ref_hybrid_export": (None, [vp, vp, vp, vp, vp, vp]),
            "ref_hybrid_spmv": (ci, [vp, vp, u64, vp, u64]),
            "ref_hybrid_free": (None, [vp]),
            "ref_run_spmv_bench": (ci, [vp, ci, i64, ci, u64, vp]),
            "ref_slabs_build": (ci, [vp, ci, u64, i64, ci, ci, pp]),
            "ref_slabs_spmv": (ci, [vp, vp, vp]),
            "ref_slabs_spmv_serial": (ci, [vp, vp, vp]),
            "ref_slabs_free": (None, [vp]),
            "ref_slabs_rgcsr_part": (ci, [vp, u64, vp, vp, vp, vp, vp]),
            "ref_slabs_count": (u64, [vp]),
            "ref_mm_parse": (ci, [C.c_char_p, u64, pp, C.POINTER(C.c_uint64)]),
            "ref_mm_write": (u64, [vp, C.c_char_p, u64]),
        }
        for k, (r, a) in sig.items():
            f = getattr(L, k)
            f.restype, f.argtypes = r, a
        _R = L
    return _R


def _rcheck(rc):
    if rc:
        msg = R().ref_last_error().decode()
        raise (ValueError if rc == 1 else RuntimeError)(msg)


class RefMatrix:
    """A reference spmvkit::TripletMatrix handle."""

    def __init__(self, h):
        self.h = C.c_void_p(h)
        r, c, n = C.c_uint64(), C.c_uint64(), C.c_uint64()
        R().ref_tm_dims(self.h, C.byref(r), C.byref(c), C.byref(n))
        self.rows, self.cols, self.nnz = r.value, c.value, n.value

    @classmethod
    def _make(cls, fn, *args):
        h = C.c_void_p()
        _rcheck(getattr(R(), fn)(*args, C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_csr(cls, m: Csr):
        return cls._make("ref_tm_from_csr", m.rows, m.cols, m.nnz, _ptr(m.rp), _ptr(m.col),
                         _ptr(m.val))

    @classmethod
    def example8(cls):
        return cls._make("ref_tm_example8")

    @classmethod
    def random_small(cls, seed, allow_zero=True, integer=True):
        return cls._make("ref_tm_random_small", seed, int(allow_zero), int(integer))

    @classmethod
    def random_case(cls, seed, max_rows):
        return cls._make("ref_tm_random_case", seed, max_rows)

    @classmethod
    def banded(cls, n, hbw, seed):
        return cls._make("ref_tm_banded", n, hbw, seed)

    def descending(self):
        return RefMatrix._make("ref_tm_descending", self.h)

    @classmethod
    def mm_parse(cls, text: bytes):
        """parse_matrix_market; returns (RefMatrix or None, error line, message)."""
        h = C.c_void_p()
        line = C.c_uint64()
        rc = R().ref_mm_parse(text, len(text), C.byref(h), C.byref(line))
        if rc:
            return None, line.value, R().ref_last_error().decode()
        return cls(h.value), 0, ""

    def mm_write(self) -> bytes:
        n = R().ref_mm_write(self.h, None, 0)
        buf = C.create_string_buffer(n)
        R().ref_mm_write(self.h, buf, n)
        return buf.raw[:n]

    def descending_map(self):
        out = np.empty(self.rows, np.uint32)
        _rcheck(R().ref_descending_map(self.h, _ptr(out)))
        return out

    def to_csr(self) -> Csr:
        rp = np.empty(self.rows + 1, np.uint32)
        col, val = np.empty(self.nnz, np.uint32), np.empty(self.nnz, np.float64)
        R().ref_tm_export(self.h, _ptr(rp), _ptr(col), _ptr(val))
        return Csr(self.rows, self.cols, rp, col, val)

    def spmv_reference(self, x):
        y = np.empty(self.rows)
        x = np.ascontiguousarray(x, np.float64)
        _rcheck(R().ref_spmv_reference(self.h, _ptr(x), x.size, _ptr(y)))
        return y

    def rgcsr(self, G, prec=8):
        h = C.c_void_p()
        _rcheck(R().ref_rgcsr_build(self.h, G, prec, C.byref(h)))
        info = np.zeros(6, np.uint64)
        R().ref_rgcsr_info(h, _ptr(info))
        slots, groups = int(info[0]), int(info[1])
        dt = np.float64 if prec == 8 else np.float32
        out = dict(values=np.empty(slots, dt), columns=np.empty(slots, np.uint32),
                   group_pointers=np.empty(groups + 1, np.uint32),
                   row_lengths=np.empty(self.rows, np.uint32), group_size=G, rows=self.rows,
                   cols=self.cols, artificial_zeros=int(info[2]), bytes_single=int(info[3]),
                   bytes_double=int(info[4]), nnz=int(info[5]), _h=h)
        R().ref_rgcsr_export(h, _ptr(out["values"]), _ptr(out["columns"]),
                             _ptr(out["group_pointers"]), _ptr(out["row_lengths"]))
        return out

    @staticmethod
    def rgcsr_spmv(a, x):
        dt = a["values"].dtype
        x = np.ascontiguousarray(x, dt)
        y = np.empty(a["rows"], dt)
        madds = C.c_uint64()
        _rcheck(R().ref_rgcsr_spmv(a["_h"], _ptr(x), x.size, _ptr(y), y.size, C.byref(madds)))
        return y, madds.value

    def hybrid(self, k1=None, prec=8):
        h = C.c_void_p()
        _rcheck(R().ref_hybrid_build(self.h, -1 if k1 is None else k1, prec, C.byref(h)))
        info = np.zeros(6, np.uint64)
        R().ref_hybrid_info(h, _ptr(info))
        k1v, es, coo = int(info[0]), int(info[1]), int(info[2])
        dt = np.float64 if prec == 8 else np.float32
        out = dict(ell_values=np.empty(es, dt), ell_columns=np.empty(es, np.uint32),
                   coo_rows=np.empty(coo, np.uint32), coo_columns=np.empty(coo, np.uint32),
                   coo_values=np.empty(coo, dt), k1=k1v, rows=self.rows, cols=self.cols,
                   artificial_zeros=int(info[3]), bytes_single=int(info[4]),
                   bytes_double=int(info[5]), _h=h)
        R().ref_hybrid_export(h, _ptr(out["ell_values"]), _ptr(out["ell_columns"]),
                              _ptr(out["coo_rows"]), _ptr(out["coo_columns"]),
                              _ptr(out["coo_values"]))
        return out

    @staticmethod
    def hybrid_spmv(h, x):
        dt = h["ell_values"].dtype
        x = np.ascontiguousarray(x, dt)
        y = np.empty(h["rows"], dt)
        _rcheck(R().ref_hybrid_spmv(h["_h"], _ptr(x), x.size, _ptr(y), y.size))
        return y

    def csr_spmv(self, x, prec=8):
        h = C.c_void_p()
        _rcheck(R().ref_csr_build(self.h, prec, C.byref(h)))
        dt = np.float64 if prec == 8 else np.float32
        x = np.ascontiguousarray(x, dt)
        y = np.empty(self.rows, dt)
        _rcheck(R().ref_csr_spmv(h, _ptr(x), x.size, _ptr(y), y.size))
        R().ref_csr_free(h)
        return y

    def __del__(self):
        if getattr(self, "h", None) and self.h.value and _R is not None:
            _R.ref_tm_free(self.h)
            self.h = C.c_void_p()


class RefSlabs:
    """The reference's own templates over group-aligned row slabs (one
    std::thread each in spmv(); in sequence in spmv_serial()), built from a
    RefMatrix: fmt 0 = spmv_csr, 1 = spmv_rgcsr (group size G), 2 =
    spmv_hybrid.  Bitwise equal to one thread (every row keeps its order)."""

    def __init__(self, ref: RefMatrix, fmt=1, G=32, prec=8, threads=None, k1=-1):
        self.h = C.c_void_p()
        self.prec, self.rows, self.cols = prec, ref.rows, ref.cols
        threads = threads or len(os.sched_getaffinity(0)) or 1
        _rcheck(R().ref_slabs_build(ref.h, fmt, G, k1, prec, threads, C.byref(self.h)))

    def _dt(self):
        return np.float64 if self.prec == 8 else np.float32

    def spmv(self, x, y=None):
        x = np.ascontiguousarray(x, self._dt())
        y = np.empty(self.rows, self._dt()) if y is None else y
        _rcheck(R().ref_slabs_spmv(self.h, _ptr(x), _ptr(y)))
        return y

    def spmv_serial(self, x, y=None):
        x = np.ascontiguousarray(x, self._dt())
        y = np.empty(self.rows, self._dt()) if y is None else y
        _rcheck(R().ref_slabs_spmv_serial(self.h, _ptr(x), _ptr(y)))
        return y

    def __len__(self):
        return int(R().ref_slabs_count(self.h))

    def rgcsr_part(self, t, arrays=True):
        """(row_begin, row_end, dict of the slab's four reference arrays)."""
        info = np.zeros(4, np.uint64)
        _rcheck(R().ref_slabs_rgcsr_part(self.h, t, _ptr(info), None, None, None, None))
        r0, r1, slots, groups = (int(v) for v in info)
        if not arrays:
            return r0, r1, {"slots": slots, "groups": groups}
        out = dict(values=np.empty(slots, self._dt()), columns=np.empty(slots, np.uint32),
                   group_pointers=np.empty(groups + 1, np.uint32),
                   row_lengths=np.empty(r1 - r0, np.uint32))
        _rcheck(R().ref_slabs_rgcsr_part(self.h, t, _ptr(info), _ptr(out["values"]),
                                         _ptr(out["columns"]), _ptr(out["group_pointers"]),
                                         _ptr(out["row_lengths"])))
        return r0, r1, out

    def free(self):
        if self.h and self.h.value and _R is not None:
            _R.ref_slabs_free(self.h)
        self.h = C.c_void_p()

    def __del__(self):
        self.free()
