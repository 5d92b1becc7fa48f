"""Host-side mirror of the reference's ``spmvkit`` hot-path API, backed by the
B200 kernels of libspmvk.so through the C-ABI (include/spmvk.h).

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/core, paths below relative to proj/):

=====================  =========================================================
this module            reference
=====================  =========================================================
TripletMatrix          spmvkit::TripletMatrix (core/include/spmvkit/triplet.hpp:26-45)
canonicalize           spmvkit::canonicalize (core/src/triplet.cpp:34-49)
row_lengths            spmvkit::row_lengths (core/src/triplet.cpp:51-55)
build_csr / spmv_csr   spmvkit/csr.hpp:24-53
build_rgcsr            spmvkit/rgcsr.hpp:38-70 (device conversion, K1)
spmv_rgcsr             spmvkit/rgcsr.hpp:72-105 (device SpMV, K2)
choose_ell_width       spmvkit/ellpack.hpp:153-166
hybrid_split_cost      spmvkit/ellpack.hpp:145-150
build_hybrid           spmvkit/ellpack.hpp:168-203
spmv_hybrid            spmvkit/ellpack.hpp:205-217
fill_report            spmvkit/fill.hpp:52-95
measured_gflops        core/src/memsim.cpp:201-207
=====================  =========================================================

``std::invalid_argument`` maps to :class:`InvalidArgument` (a ``ValueError``),
``std::runtime_error`` to :class:`SpmvkRuntimeError`.  x / y may be numpy
arrays (host span semantics: H2D, SpMV, D2H, synchronous) or CUDA torch
tensors (device-resident; launched on torch's current stream).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Iterable, Optional

import numpy as np

from . import _lib
from ._lib import F32, F64, HybridInfo, RgcsrInfo, lib


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class SpmvkRuntimeError(RuntimeError):
    """std::runtime_error in the reference (size budgets, 32-bit overflow)."""


class CudaError(RuntimeError):
    """Device / launch failure (no CPU fallback exists)."""


def _check(rc: int) -> None:
    if rc == _lib.SPMVK_OK:
        return
    msg = _lib.last_error()
    if rc == _lib.SPMVK_EINVAL:
        raise InvalidArgument(msg)
    if rc == _lib.SPMVK_ERANGE:
        raise SpmvkRuntimeError(msg)
    raise CudaError(f"spmvk status {rc}: {msg}")


def _prec(p) -> int:
    if p in (F32, "f32", "float32", "single", np.float32):
        return F32
    if p in (F64, "f64", "float64", "double", np.float64, None):
        return F64
    raise InvalidArgument(f"unknown precision {p!r}")


def _dtype(prec: int):
    return np.float32 if prec == F32 else np.float64


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data if a.size else 0


# ---------------------------------------------------------------- data model
class TripletMatrix:
    """Canonical coordinate matrix held as CSR arrays on the host.

    A canonical TripletMatrix (entries strictly increasing in (row, col)) is
    exactly a CSR matrix whose k-th entry is the k-th sorted triplet; the
    constructor validates like the reference's (src/triplet.cpp:22-32).
    """

    def __init__(self, num_rows: int, num_cols: int, row_ptr, col, val, validate=True):
        self.num_rows = int(num_rows)
        self.num_cols = int(num_cols)
        self.row_ptr = np.ascontiguousarray(row_ptr, dtype=np.uint32)
        self.col = np.ascontiguousarray(col, dtype=np.uint32)
        self.val = np.ascontiguousarray(val, dtype=np.float64)
        if validate:
            self._validate()

    def _validate(self):
        rp, n = self.row_ptr, self.num_rows
        if rp.shape != (n + 1,) or rp[0] != 0 or rp[-1] != self.col.size or \
                self.col.size != self.val.size or np.any(np.diff(rp.astype(np.int64)) < 0):
            raise InvalidArgument("row pointers are not a monotone offset array ending at nnz")
        if self.col.size and int(self.col.max()) >= self.num_cols:
            raise InvalidArgument("entry outside the matrix")
        if self.col.size > 1:
            rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp.astype(np.int64)))
            same = rows[1:] == rows[:-1]
            if np.any(same & (self.col[1:] <= self.col[:-1])):
                raise InvalidArgument("entries not strictly increasing in (row, col)")

    @classmethod
    def from_entries(cls, num_rows: int, num_cols: int, entries: Iterable):
        """TripletMatrix(num_rows, num_cols, {{row, col, value}, ...})."""
        e = list(entries)
        rows = np.array([t[0] for t in e], dtype=np.int64)
        for t in e:
            if t[0] >= num_rows or t[1] >= num_cols or t[0] < 0 or t[1] < 0:
                raise InvalidArgument(f"entry ({t[0]}, {t[1]}) outside {num_rows}x{num_cols} matrix")
        rp = np.zeros(num_rows + 1, dtype=np.int64)
        np.add.at(rp, rows + 1, 1)
        if len(e) > 1 and any((a[0], a[1]) >= (b[0], b[1]) for a, b in zip(e, e[1:])):
            raise InvalidArgument("entries not strictly increasing in (row, col)")
        return cls(num_rows, num_cols, np.cumsum(rp), [t[1] for t in e], [t[2] for t in e])

    @property
    def nnz(self) -> int:
        return int(self.col.size)

    def entries(self):
        rows = np.repeat(np.arange(self.num_rows), np.diff(self.row_ptr.astype(np.int64)))
        return list(zip(rows.tolist(), self.col.tolist(), self.val.tolist()))


def canonicalize(raw: Iterable, num_rows: int, num_cols: int) -> TripletMatrix:
    """Sorts by (row, col) and sums duplicates (src/triplet.cpp:34-49)."""
    e = list(raw)
    for t in e:
        if t[0] >= num_rows or t[1] >= num_cols:
            raise InvalidArgument(f"entry ({t[0]}, {t[1]}) outside {num_rows}x{num_cols} matrix")
    e.sort(key=lambda t: (t[0], t[1]))  # stable, as std::sort ties do not matter after merging
    merged = []
    for t in e:
        if merged and merged[-1][0] == t[0] and merged[-1][1] == t[1]:
            merged[-1][2] += t[2]
        else:
            merged.append([t[0], t[1], float(t[2])])
    return TripletMatrix.from_entries(num_rows, num_cols, merged)


def row_lengths(m: TripletMatrix) -> np.ndarray:
    return np.diff(m.row_ptr.astype(np.int64)).astype(np.uint64)


# ---------------------------------------------------------------- CSR (device)
def _release(obj, destroy: str):
    """Frees a handle from __del__; a no-op once interpreter shutdown has torn
    down this module's globals (the library may already be unloaded)."""
    try:
        h = getattr(obj, "_h", None)
        lib_mod = _lib
        if not h or not h.value or lib_mod is None or getattr(lib_mod, "_lib", None) is None:
            return
        getattr(lib_mod._lib, destroy)(h)
        obj._h = C.c_void_p()
    except Exception:  # noqa: BLE001 -- never raise from a finalizer
        pass


class CsrMatrix:
    """Device CSR (build_csr's CsrMatrix, csr.hpp:13-22) owned by a handle."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        r, c, n, p = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_int()
        _check(lib().spmvk_csr_shape(self._h, C.byref(r), C.byref(c), C.byref(n), C.byref(p)))
        self.num_rows, self.num_cols, self._nnz, self.val_prec = r.value, c.value, n.value, p.value

    def nnz(self) -> int:
        return self._nnz

    @classmethod
    def stencil(cls, kind: int, n: int, stream: int = 0) -> "CsrMatrix":
        """5-/7-/27-point stencil generated directly in HBM."""
        h = C.c_void_p()
        _check(lib().spmvk_csr_stencil(kind, n, stream or None, C.byref(h)))
        return cls(h.value)

    def to_host(self):
        rp = np.empty(self.num_rows + 1, np.uint32)
        col = np.empty(self._nnz, np.uint32)
        val = np.empty(self._nnz, _dtype(self.val_prec))
        _check(lib().spmvk_csr_download(self._h, _ptr(rp), _ptr(col), _ptr(val)))
        return rp, col, val

    def row_length_range(self):
        out = (C.c_uint64 * 2)()
        _check(lib().spmvk_csr_row_length_range(self._h, out))
        return int(out[0]), int(out[1])

    def __del__(self, _release=_release):  # bound now: module globals vanish at exit
        _release(self, "spmvk_csr_destroy")


class MatrixMarketError(RuntimeError):
    """spmvkit::MatrixMarketError (matrix_market.hpp:14-23): message "line N: ..."
    and the 1-based line number in ``.line``."""

    def __init__(self, message: str, line: int):
        super().__init__(message)
        self.line = line


def _mm_check(rc: int, line: C.c_uint64) -> None:
    if rc == _lib.SPMVK_EPARSE:
        raise MatrixMarketError(_lib.last_error(), line.value)
    _check(rc)


def parse_matrix_market(text, precision=F64, threads: int = 0, stream: int = 0) -> CsrMatrix:
    """parse_matrix_market (src/matrix_market.cpp:61-138) straight to a device
    CSR: same accepted language, messages and line numbers; canonicalised."""
    data = text.encode() if isinstance(text, str) else bytes(text)
    h = C.c_void_p()
    line = C.c_uint64()
    _mm_check(lib().spmvk_mm_parse(data, len(data), threads, _prec(precision), stream or None,
                                   C.byref(h), C.byref(line)), line)
    return CsrMatrix(h.value)


def load_matrix_market(path, precision=F64, threads: int = 0, stream: int = 0) -> CsrMatrix:
    """load_matrix_market (src/matrix_market.cpp:140-148); parse errors carry
    the path prefix like the reference's rethrow."""
    h = C.c_void_p()
    line = C.c_uint64()
    _mm_check(lib().spmvk_mm_load(str(path).encode(), threads, _prec(precision), stream or None,
                                  C.byref(h), C.byref(line)), line)
    return CsrMatrix(h.value)


def write_matrix_market(a, threads: int = 0) -> str:
    """write_matrix_market (src/matrix_market.cpp:150-158) of a CSR handle (or
    anything build_csr accepts): the reference's text byte for byte."""
    a = _as_csr(a)
    n = C.c_uint64()
    _check(lib().spmvk_mm_write(a._h, threads, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(lib().spmvk_mm_write(a._h, threads, buf, n.value, C.byref(n)))
    return buf.raw[: n.value].decode()


def save_matrix_market(path, a, threads: int = 0) -> None:
    """save_matrix_market (src/matrix_market.cpp:160-164)."""
    a = _as_csr(a)
    _check(lib().spmvk_mm_save(a._h, str(path).encode(), threads))


@dataclass
class MatrixStats:
    """spmvkit::MatrixStats (triplet.hpp:54-61)."""
    num_rows: int
    nnz: int
    row_len_max: int
    row_len_mean: float
    row_len_min: int
    density_percent: float


def matrix_stats(m) -> MatrixStats:
    """matrix_stats (src/triplet.cpp:57-69); row-length extremes from the device."""
    a = _as_csr(m)
    if a.num_rows == 0:
        raise InvalidArgument("matrix_stats: matrix has zero rows")
    mx, mn = a.row_length_range()
    nnz = a.nnz()
    cells = float(a.num_rows) * float(a.num_cols)
    return MatrixStats(a.num_rows, nnz, mx, nnz / a.num_rows, mn,
                       100.0 * nnz / cells if cells > 0 else 0.0)


def descending_row_permutation(m) -> np.ndarray:
    """descending_row_permutation(m) (src/reorder.cpp:35-42) on the device:
    map[new] = old, rows by decreasing length, ties by original index."""
    a = _as_csr(m)
    out = np.empty(a.num_rows, np.uint32)
    _check(lib().spmvk_csr_descending_permutation(a._h, _ptr(out)))
    return out


def apply_descending_permutation(m, stream: int = 0):
    """apply_permutation(m, descending_row_permutation(m), RowsOnly)
    (src/reorder.cpp:44-61) on the device.  Returns (CsrMatrix, map); row i of
    the result is row map[i] of m, so spmv(result, x)[i] == spmv(m, x)[map[i]]."""
    a = _as_csr(m)
    out = np.empty(a.num_rows, np.uint32)
    h = C.c_void_p()
    _check(lib().spmvk_csr_permute_rows_descending(a._h, stream or None, C.byref(h), _ptr(out)))
    return CsrMatrix(h.value), out


class Permutation:
    """spmvkit::Permutation (reorder.hpp, src/reorder.cpp:12-33): a bijection
    map[new] = old on 0..n-1, validated on construction."""

    def __init__(self, mapping):
        self._map = np.ascontiguousarray(mapping, dtype=np.int64)
        n = self._map.size
        ok = bool(((self._map >= 0) & (self._map < n)).all()) if n else True
        if not ok or (n and np.bincount(self._map, minlength=n).max() > 1):
            raise InvalidArgument(f"permutation is not a bijection on 0..{n - 1 if n else 0}")
        self._map = self._map.astype(np.uint32)
        self._dev = None

    @classmethod
    def identity(cls, n: int) -> "Permutation":
        return cls(np.arange(n, dtype=np.uint32))

    def map(self) -> np.ndarray:
        return self._map

    def size(self) -> int:
        return int(self._map.size)

    def __len__(self) -> int:
        return self.size()

    def __getitem__(self, i):
        return self._map[i]

    def inverse(self) -> np.ndarray:
        inv = np.empty_like(self._map)
        inv[self._map] = np.arange(self._map.size, dtype=np.uint32)
        return inv

    def device_map(self):
        """The map as a CUDA uint32 buffer (cached)."""
        if self._dev is None:
            import torch
            self._dev = torch.from_numpy(self._map.view(np.int32)).cuda()
        return self._dev


def parse_permutation(text: str) -> Permutation:
    """parse_permutation (src/reorder.cpp:63-85): one 0-based index per line,
    blank lines skipped, the reference's messages."""
    out = []
    for no, line in enumerate(text.split("\n"), 1):
        if line.endswith("\r"):
            line = line[:-1]
        if not line.strip(" \t"):
            continue
        s = line.lstrip(" \t\n\v\f\r")
        j = 1 if s[:1] in "+-" else 0
        while j < len(s) and s[j].isdigit():
            j += 1
        if j == 0 or not s[:j].lstrip("+-"):
            raise InvalidArgument(f"permutation line {no}: expected an index, got '{line}'")
        v = int(s[:j])
        if v < 0 or s[j:].strip(" \t"):
            raise InvalidArgument(
                f"permutation line {no}: expected a single 0-based index, got '{line}'")
        out.append(v)
    return Permutation(np.array(out, dtype=np.int64))


def load_permutation(path) -> Permutation:
    """load_permutation (src/reorder.cpp:87-91)."""
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise SpmvkRuntimeError(f"cannot open {path}") from None
    return parse_permutation(text)


def apply_permutation(m, p, mode: str = "rows_only", stream: int = 0) -> CsrMatrix:
    """apply_permutation(m, p, RowsOnly | Symmetric) (src/reorder.cpp:44-61) on
    the device: row i of the result is row p[i] of m; "symmetric" also
    relabels the columns (square matrices) and re-sorts each row."""
    if mode not in ("rows_only", "symmetric"):
        raise InvalidArgument(f"unknown permutation mode {mode!r}")
    p = p if isinstance(p, Permutation) else Permutation(p)
    a = _as_csr(m)
    h = C.c_void_p()
    mp = p.map()
    _check(lib().spmvk_csr_permute(a._h, _ptr(mp) if mp.size else None, mp.size,
                                   1 if mode == "symmetric" else 0, stream or None, C.byref(h)))
    return CsrMatrix(h.value)


def permute_vector(p: Permutation, v, inverse: bool = False, stream: Optional[int] = None):
    """out[i] = v[p[i]] (into the permuted numbering), or with inverse=True
    out[p[i]] = v[i] (a permuted matrix's y back to the original row order).
    CUDA tensors in and out."""
    import torch
    if not (_is_torch(v) and v.is_cuda and v.is_contiguous()):
        raise InvalidArgument("permute_vector takes a contiguous CUDA tensor")
    if v.numel() != p.size():
        raise InvalidArgument("permute_vector: vector length differs from the permutation")
    out = torch.empty_like(v)
    fn = {torch.float64: lib().spmvk_permute_vector_f64,
          torch.float32: lib().spmvk_permute_vector_f32}.get(v.dtype)
    if fn is None:
        raise InvalidArgument("permute_vector: float32 or float64 vectors")
    s = stream if stream is not None else _torch_stream(v)
    _check(fn(p.device_map().data_ptr() if p.size() else None, p.size(), v.data_ptr(),
              out.data_ptr(), 1 if inverse else 0, s or None))
    return out


def build_csr(m: TripletMatrix, precision=F64, stream: int = 0) -> CsrMatrix:
    """build_csr<Scalar>(m) (csr.hpp:24-39): upload + validate on the device."""
    prec = _prec(precision)
    val = m.val if prec == F64 else m.val.astype(np.float32)
    h = C.c_void_p()
    _check(lib().spmvk_csr_upload(m.num_rows, m.num_cols, m.nnz, _ptr(m.row_ptr), _ptr(m.col),
                                  _ptr(val), prec, stream or None, C.byref(h)))
    return CsrMatrix(h.value)


def _as_csr(m) -> CsrMatrix:
    if isinstance(m, CsrMatrix):
        return m
    if isinstance(m, TripletMatrix):
        return build_csr(m, F64)
    raise InvalidArgument(f"expected TripletMatrix or CsrMatrix, got {type(m).__name__}")


# ---------------------------------------------------------------- SpMV plumbing
def _is_torch(t) -> bool:
    return type(t).__module__.startswith("torch")


def _torch_stream(t) -> int:
    import torch
    return torch.cuda.current_stream(t.device).cuda_stream


def _device_call(fn_name_prefix: str, handle, x, y, n_rows: int, n_cols: int, prec: int,
                 stream: Optional[int]):
    import torch
    dt = torch.float32 if prec == F32 else torch.float64
    if not (x.is_cuda and x.is_contiguous()):
        raise InvalidArgument("x must be a contiguous CUDA tensor")
    if y is None:
        y = torch.empty(n_rows, dtype=dt, device=x.device)
    if x.dtype != dt or y.dtype != dt:
        raise InvalidArgument(f"{fn_name_prefix}: handle precision differs from the x/y dtype")
    s = stream if stream is not None else _torch_stream(x)
    sfx = "f32" if prec == F32 else "f64"
    _check(getattr(lib(), f"{fn_name_prefix}_{sfx}")(handle, x.data_ptr(), x.numel(),
                                                     y.data_ptr(), y.numel(), s or None))
    return y


# ---------------------------------------------------------------- RgCSR
@dataclass
class FillReport:
    """spmvkit::FillReport (fill.hpp:18-26)."""
    format_name: str
    stored_slots: int
    nnz: int
    artificial_zeros: int
    fill_percent: float
    bytes_single: int
    bytes_double: int


def _fill_percent(az: int, nnz: int) -> float:
    return 0.0 if nnz == 0 else 100.0 * az / nnz


class RgcsrMatrix:
    """Device RgCSR (RgcsrMatrix<S>, rgcsr.hpp:19-36) owned by a handle."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        self.info = RgcsrInfo()
        _check(lib().spmvk_rgcsr_get_info(self._h, C.byref(self.info)))
        self.num_rows = self.info.num_rows
        self.num_cols = self.info.num_cols
        self.group_size = self.info.group_size
        self.precision = self.info.precision

    def num_groups(self) -> int:
        return self.info.num_groups

    def rows_in_group(self, g: int) -> int:
        return min(self.group_size, self.num_rows - g * self.group_size)

    def slot_count(self) -> int:
        return self.info.slots

    def nnz(self) -> int:
        return self.info.nnz

    def to_host(self) -> dict:
        """The four reference arrays: values, columns, group_pointers, row_lengths."""
        i = self.info
        out = dict(values=np.empty(i.slots, _dtype(self.precision)),
                   columns=np.empty(i.slots, np.uint32),
                   group_pointers=np.empty(i.num_groups + 1, np.uint32),
                   row_lengths=np.empty(i.num_rows, np.uint32))
        _check(lib().spmvk_rgcsr_download(self._h, _ptr(out["values"]), _ptr(out["columns"]),
                                          _ptr(out["group_pointers"]), _ptr(out["row_lengths"])))
        return out

    def __del__(self, _release=_release):  # bound now: module globals vanish at exit
        _release(self, "spmvk_rgcsr_destroy")


def build_rgcsr(m, group_size: int, precision=F64, stream: int = 0,
                row_range: Optional[tuple] = None) -> RgcsrMatrix:
    """build_rgcsr<S>(m, group_size) (rgcsr.hpp:38-70) on the device.

    ``m`` is a TripletMatrix (uploaded first) or a device CsrMatrix.  Raises
    InvalidArgument for group_size == 0 (the reference's message) and
    SpmvkRuntimeError when the slot count overflows uint32 (the reference
    truncates silently, rgcsr.hpp:56).  ``row_range=(r0, r1)`` builds the
    group-aligned row slab used by the partitioner.
    """
    if group_size < 0:
        raise InvalidArgument("build_rgcsr: group size must be nonzero")
    a = _as_csr(m)
    h = C.c_void_p()
    if row_range is None:
        _check(lib().spmvk_rgcsr_build(a._h, group_size, _prec(precision), stream or None,
                                       C.byref(h)))
    else:
        _check(lib().spmvk_rgcsr_build_rows(a._h, row_range[0], row_range[1], group_size,
                                            _prec(precision), stream or None, C.byref(h)))
    return RgcsrMatrix(h.value)


class _HostBuffer:
    """Owner of one spmvk_host_alloc block; numpy arrays over it keep it alive."""

    def __init__(self, ptr: int, nbytes: int, dtype: np.dtype, n: int):
        self.ptr = ptr
        self.__array_interface__ = {"shape": (n,), "typestr": dtype.str, "version": 3,
                                    "data": (ptr, False)}

    def __del__(self):
        if self.ptr:
            try:
                lib().spmvk_host_free(C.c_void_p(self.ptr))
            except Exception:  # noqa: BLE001 -- interpreter shutdown: the OS reclaims it
                pass
            self.ptr = 0


def host_array(n: int, dtype=np.float64) -> np.ndarray:
    """A zeroed numpy array on page-locked 2 MB-page host memory
    (spmvk_host_alloc) for the span overloads' x and y; freed when the last
    array over it is collected.  Any pinned buffer works for the pipelined
    host-span path; this one avoids the slow first calls of freshly pinned
    4 KB pages (profiles/r02t_e2e_env.md)."""
    dt = np.dtype(dtype)
    p = C.c_void_p()
    _check(lib().spmvk_host_alloc(max(1, n * dt.itemsize), C.byref(p)))
    return np.asarray(_HostBuffer(p.value, n * dt.itemsize, dt, n))


def spmv_rgcsr(a: RgcsrMatrix, x, y=None, multiply_add_count: bool = False,
               stream: Optional[int] = None):
    """spmv_rgcsr(a, x[, y][, &madds]) (rgcsr.hpp:75-105).

    numpy x -> host span semantics (returns numpy y, plus the multiply-add
    count when requested); CUDA tensor x -> device-resident launch on the
    current stream (returns the y tensor)."""
    if _is_torch(x):
        y = _device_call("spmvk_rgcsr_spmv", a._h, x, y, a.num_rows, a.num_cols, a.precision,
                         stream)
        return (y, a.nnz()) if multiply_add_count else y
    dt = _dtype(a.precision)
    x = np.ascontiguousarray(x)
    if x.dtype != dt:
        raise InvalidArgument("spmv_rgcsr: handle precision differs from the x dtype")
    if y is None:
        y = np.empty(a.num_rows, dt)
    madds = C.c_uint64()
    fn = lib().spmvk_rgcsr_spmv_host_f32 if a.precision == F32 else lib().spmvk_rgcsr_spmv_host_f64
    _check(fn(a._h, _ptr(x), x.size, _ptr(y), y.size, C.byref(madds)))
    return (y, madds.value) if multiply_add_count else y


def persist_x(x, stream: Optional[int] = None, hit_ratio: float = 1.0) -> int:
    """L2 persistence window over the CUDA tensor ``x`` for kernels launched on
    ``stream`` (default: torch's current stream) -- spmvk_stream_persist_x.
    Returns the persisting-L2 carve-out granted in bytes; ``x=None`` resets."""
    import torch
    if stream is None:
        stream = torch.cuda.current_stream().cuda_stream
    g = C.c_uint64()
    if x is None:
        _check(lib().spmvk_stream_persist_x(C.c_void_p(stream), None, 0, 1.0, C.byref(g)))
    else:
        _check(lib().spmvk_stream_persist_x(C.c_void_p(stream), C.c_void_p(x.data_ptr()),
                                            x.numel() * x.element_size(), hit_ratio, C.byref(g)))
    return g.value


# ---------------------------------------------------------------- Hybrid
def hybrid_split_cost(row_lens, k: int) -> int:
    """hybrid_split_cost (ellpack.hpp:145-150)."""
    L = np.ascontiguousarray(row_lens, dtype=np.uint64)
    return int(lib().spmvk_hybrid_split_cost(_ptr(L), L.size, k))


def choose_ell_width(row_lens) -> int:
    """choose_ell_width (ellpack.hpp:153-166): histogram + suffix sums."""
    L = np.ascontiguousarray(row_lens, dtype=np.uint64)
    return int(lib().spmvk_choose_ell_width(_ptr(L), L.size))


class HybridMatrix:
    """Device Hybrid ELL+COO (HybridMatrix<S>, ellpack.hpp:44-48)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        self.info = HybridInfo()
        _check(lib().spmvk_hybrid_get_info(self._h, C.byref(self.info)))
        self.num_rows = self.info.num_rows
        self.num_cols = self.info.num_cols
        self.precision = self.info.precision

    @property
    def slots_per_row(self) -> int:
        return self.info.ell_width

    def coo_nnz(self) -> int:
        return self.info.coo_nnz

    def to_host(self) -> dict:
        i, dt = self.info, _dtype(self.precision)
        out = dict(ell_values=np.empty(i.ell_slots, dt), ell_columns=np.empty(i.ell_slots, np.uint32),
                   coo_rows=np.empty(i.coo_nnz, np.uint32), coo_columns=np.empty(i.coo_nnz, np.uint32),
                   coo_values=np.empty(i.coo_nnz, dt))
        _check(lib().spmvk_hybrid_download(self._h, *(_ptr(out[k]) for k in (
            "ell_values", "ell_columns", "coo_rows", "coo_columns", "coo_values"))))
        return out

    def __del__(self, _release=_release):  # bound now: module globals vanish at exit
        _release(self, "spmvk_hybrid_destroy")


def build_hybrid(m, k1: Optional[int] = None, precision=F64, stream: int = 0) -> HybridMatrix:
    """build_hybrid<S>(m, k1) (ellpack.hpp:168-203); k1=None chooses the width."""
    a = _as_csr(m)
    h = C.c_void_p()
    _check(lib().spmvk_hybrid_build(a._h, -1 if k1 is None else int(k1), _prec(precision),
                                    stream or None, C.byref(h)))
    return HybridMatrix(h.value)


K_DEFAULT_ELL_SLOT_BUDGET = 1 << 31  # kDefaultEllSlotBudget (ellpack.hpp:80)


def build_ellpack(m, slot_budget: int = K_DEFAULT_ELL_SLOT_BUDGET, precision=F64,
                  stream: int = 0) -> HybridMatrix:
    """build_ellpack<S>(m, slot_budget) (ellpack.hpp:84-107): ELLPACK of width
    K = max row length (a Hybrid handle without COO, fill_report "ellpack").
    Raises SpmvkRuntimeError (std::runtime_error) past the slot budget."""
    a = _as_csr(m)
    h = C.c_void_p()
    _check(lib().spmvk_ellpack_build(a._h, int(slot_budget), _prec(precision), stream or None,
                                     C.byref(h)))
    return HybridMatrix(h.value)


def _hybrid_part(fn: str, h: HybridMatrix, x, y, stream, need_y: bool):
    if _is_torch(x):
        if need_y and y is None:
            raise InvalidArgument(f"{fn}: y is required (it accumulates)")
        return _device_call(f"spmvk_hybrid_{fn}", h._h, x, y, h.num_rows, h.num_cols,
                            h.precision, stream)
    dt = _dtype(h.precision)
    x = np.ascontiguousarray(x)
    if x.dtype != dt:
        raise InvalidArgument(f"{fn}: handle precision differs from the x dtype")
    if y is None:
        if need_y:
            raise InvalidArgument(f"{fn}: y is required (it accumulates)")
        y = np.empty(h.num_rows, dt)
    if not (isinstance(y, np.ndarray) and y.dtype == dt and y.flags.c_contiguous):
        raise InvalidArgument(f"{fn}: y must be a contiguous array of the handle precision")
    sfx = "f32" if h.precision == F32 else "f64"
    _check(getattr(lib(), f"spmvk_hybrid_{fn}_host_{sfx}")(h._h, _ptr(x), x.size, _ptr(y),
                                                           y.size))
    return y


def spmv_ellpack(h: HybridMatrix, x, y=None, stream: Optional[int] = None):
    """spmv_ellpack(h.ell, x, y) (ellpack.hpp:110-130): the ELL part only."""
    return _hybrid_part("spmv_ell", h, x, y, stream, need_y=False)


def spmv_coo(h: HybridMatrix, x, y, stream: Optional[int] = None):
    """spmv_coo(h.coo, x, y) (ellpack.hpp:132-141): y[row] += v * x[col] over
    the COO part in array order, in place."""
    return _hybrid_part("spmv_coo", h, x, y, stream, need_y=True)


def spmv_hybrid(h: HybridMatrix, x, y=None, stream: Optional[int] = None):
    """spmv_hybrid(h, x, y) (ellpack.hpp:205-217)."""
    if _is_torch(x):
        return _device_call("spmvk_hybrid_spmv", h._h, x, y, h.num_rows, h.num_cols,
                            h.precision, stream)
    dt = _dtype(h.precision)
    x = np.ascontiguousarray(x)
    if x.dtype != dt:
        raise InvalidArgument("spmv_hybrid: handle precision differs from the x dtype")
    if y is None:
        y = np.empty(h.num_rows, dt)
    fn = lib().spmvk_hybrid_spmv_host_f32 if h.precision == F32 else lib().spmvk_hybrid_spmv_host_f64
    _check(fn(h._h, _ptr(x), x.size, _ptr(y), y.size))
    return y


def spmv_csr(a: CsrMatrix, x, y=None, stream: Optional[int] = None):
    """spmv_csr(a, x, y) (csr.hpp:41-53), device tensors only."""
    if not _is_torch(x):
        raise InvalidArgument("spmv_csr on the device takes CUDA tensors")
    return _device_call("spmvk_csr_spmv", a._h, x, y, a.num_rows, a.num_cols, a.val_prec, stream)


# ---------------------------------------------------------------- CG (§8f-4)
def cg(a: RgcsrMatrix, b, x0=None, tol: float = 1e-10, max_iter: int = 1000,
       check_every: int = 10, stream: Optional[int] = None):
    """Conjugate gradients on the device for an SPD fp64 RgCSR matrix (the
    paper's motivating workload; not in the reference).  b (and x0) are CUDA
    float64 tensors.  Returns (x, iterations, relative residual)."""
    import torch
    if a.precision != F64:
        raise InvalidArgument("cg: fp64 RgCSR required")
    x = torch.zeros_like(b) if x0 is None else x0.clone()
    it = C.c_uint64()
    res = C.c_double()
    s = stream if stream is not None else _torch_stream(b)
    _check(lib().spmvk_cg_solve_f64(a._h, b.data_ptr(), x.data_ptr(), b.numel(), tol, max_iter,
                                    check_every, C.byref(it), C.byref(res), s or None))
    return x, it.value, res.value


def to_triplets(a) -> TripletMatrix:
    """to_triplets for RgCSR (rgcsr.hpp:107-123), Hybrid (ellpack.hpp:219-240)
    and device CSR (csr.hpp:62-72): the canonical host TripletMatrix."""
    if isinstance(a, CsrMatrix):
        c = a
    else:
        h = C.c_void_p()
        fn = lib().spmvk_rgcsr_to_csr if isinstance(a, RgcsrMatrix) else lib().spmvk_hybrid_to_csr
        _check(fn(a._h, None, C.byref(h)))
        c = CsrMatrix(h.value)
    rp, col, val = c.to_host()
    return TripletMatrix(c.num_rows, c.num_cols, rp, col, val.astype(np.float64))


# ---------------------------------------------------------------- accounting
def fill_report(a) -> FillReport:
    """fill_report (fill.hpp:52-95) for CSR, RgCSR, ELLPACK and Hybrid handles."""
    i = getattr(a, "info", None)
    if isinstance(a, RgcsrMatrix):
        return FillReport("rgcsr", i.slots, i.nnz, i.artificial_zeros,
                          _fill_percent(i.artificial_zeros, i.nnz), i.bytes_single, i.bytes_double)
    if isinstance(a, CsrMatrix):  # fill_report(CsrMatrix) (fill.hpp:52-55)
        n = a.nnz()
        words = n + a.num_rows + 1
        return FillReport("csr", n, n, 0, 0.0, n * 4 + words * 4, n * 8 + words * 4)
    if isinstance(a, HybridMatrix) and i.ellpack:
        # fill_report(EllpackMatrix) (fill.hpp:61-64): nnz = ell_nnz recount, words = slots
        az = i.ell_slots - i.fill_nnz
        return FillReport("ellpack", i.ell_slots, i.fill_nnz, az, _fill_percent(az, i.fill_nnz),
                          i.ell_slots * 8, i.ell_slots * 12)
    if isinstance(a, HybridMatrix):
        # the reference recounts ELL nnz from the layout (ell_nnz, ellpack.hpp:55-78)
        return FillReport("hybrid", i.ell_slots + i.coo_nnz, i.fill_nnz, i.artificial_zeros,
                          _fill_percent(i.artificial_zeros, i.fill_nnz), i.bytes_single,
                          i.bytes_double)
    raise InvalidArgument(f"no fill report for {type(a).__name__}")


B200_COPY_GBS = 6545.3  # MEASURED_PEAKS.json hbm_gbs on this pool's B200s


@dataclass
class PeakEstimate:
    """spmvkit::PeakEstimate (memsim.hpp:92-99)."""
    precision: str
    cached_x: bool
    bytes_per_nnz: int
    gflops: float


def peak_performance(precision=F64, cached_x: bool = True,
                     bandwidth_gb_s: float = B200_COPY_GBS, index_bytes: int = 4) -> PeakEstimate:
    """peak_performance (memsim.cpp:192-199): 2 * BW / (index + S * (cached ? 1 : 2))
    flops per byte-bound SpMV, for the B200's measured bandwidth by default
    (the reference's AccessModel defaults to a GTX 280, 141.7 GB/s)."""
    sv = _prec(precision)
    bpn = index_bytes + sv * (1 if cached_x else 2)
    return PeakEstimate("double" if sv == F64 else "single", bool(cached_x), bpn,
                        2.0 * bandwidth_gb_s / bpn)


def measured_gflops(nnz: int, seconds: float) -> float:
    """2 * nnz / seconds / 1e9 (memsim.cpp:201-207)."""
    if not seconds > 0.0:
        raise InvalidArgument(f"measured_gflops: seconds must be positive, got {seconds}")
    return 2.0 * nnz / seconds / 1e9


# ---------------------------------------------------------------- bench harness
class ChecksumError(RuntimeError):
    """spmvkit::ChecksumError (bench.hpp:33-37): a format disagrees with the oracle."""


FORMAT_KINDS = ("csr", "ellpack", "coo", "hybrid", "bcsr", "rgcsr")  # format_kind.hpp


@dataclass
class BenchOptions:
    """spmvkit::BenchOptions (bench.hpp:39-44)."""
    repetitions: int = 20
    x_ones: bool = False
    seed: int = 1
    target_rep_seconds: float = 2e-4


@dataclass
class BenchRecord:
    """spmvkit::BenchRecord (bench.hpp:16-29)."""
    matrix_name: str
    format_name: str
    group_size: Optional[int]
    precision: str
    repetitions: int
    nnz: int
    median_seconds: float
    gflops: float
    fill_percent: float
    artificial_zeros: int
    bytes: int
    checksum: float


def run_spmv_bench(m: TripletMatrix, matrix_name: str, kind: str, group_size: Optional[int] = None,
                   precision=F64, options: Optional[BenchOptions] = None) -> BenchRecord:
    """run_spmv_bench (src/bench.cpp:47-138) on the B200: builds the format on
    the device, gates the y checksum against spmv_reference on the
    storage-quantized inputs (the fp64 device CSR SpMV: same sorted-entry
    accumulation; tolerance 1e-10 fp64 / 1e-5 fp32 relative), then reports the
    median of `repetitions` device-timed repetitions, each a calibrated
    inner loop of at least `target_rep_seconds` (CUDA events; A, x and y stay
    resident in HBM -- the device analogue of the reference's host arrays)."""
    import torch
    o = options or BenchOptions()
    prec = _prec(precision)
    if kind not in FORMAT_KINDS:
        raise InvalidArgument(f"unknown format {kind!r}")
    if kind == "coo":
        raise InvalidArgument("run_spmv_bench: coo is benchmarked as part of hybrid")
    if kind == "bcsr":
        raise InvalidArgument("run_spmv_bench: bcsr is not on the B200 path")
    dt_np = np.float32 if prec == F32 else np.float64
    dt = torch.float32 if prec == F32 else torch.float64
    if o.x_ones:
        xd = np.ones(m.num_cols)
    else:
        xd = np.empty(m.num_cols)
        lib().spmvk_gen_random_vector(m.num_cols, o.seed, _ptr(xd))
    x = torch.from_numpy(xd.astype(dt_np)).cuda()
    y = torch.zeros(m.num_rows, dtype=dt, device="cuda")
    # oracle inputs: values and x quantized to the storage precision, in fp64
    q = TripletMatrix(m.num_rows, m.num_cols, m.row_ptr, m.col,
                      m.val.astype(dt_np).astype(np.float64), validate=False)
    y_ref = spmv_csr(build_csr(q, F64), x.double())
    if kind == "csr":
        a = build_csr(m, prec)
        fn = lambda: spmv_csr(a, x, y)  # noqa: E731
    elif kind == "ellpack":
        a = build_ellpack(m, precision=prec)
        fn = lambda: spmv_ellpack(a, x, y)  # noqa: E731
    elif kind == "hybrid":
        a = build_hybrid(m, group_size, prec)
        fn = lambda: spmv_hybrid(a, x, y)  # noqa: E731
    else:
        a = build_rgcsr(m, group_size if group_size is not None else 32, prec)
        fn = lambda: spmv_rgcsr(a, x, y)  # noqa: E731
    fill = fill_report(a)
    fn()
    # sequential sums in row order, as the reference's loops (bench.cpp:106-109)
    checksum = float(np.cumsum(y.double().cpu().numpy())[-1]) if m.num_rows else 0.0
    checksum_ref = float(np.cumsum(y_ref.cpu().numpy())[-1]) if m.num_rows else 0.0
    tol = 1e-10 if prec == F64 else 1e-5
    if abs(checksum - checksum_ref) > tol * max(1.0, abs(checksum_ref)):
        raise ChecksumError(f"{kind} checksum {checksum:.6f} disagrees with oracle "
                            f"{checksum_ref:.6f} on {matrix_name}")

    def time_once(inner: int) -> float:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(inner):
            fn()
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) * 1e-3 / inner

    inner = 1
    probe = time_once(inner)
    while probe * inner < o.target_rep_seconds and inner < (1 << 20):
        inner *= 8
        probe = time_once(inner)
    times = sorted(time_once(inner) for _ in range(max(o.repetitions, 1)))
    med = times[len(times) // 2]
    return BenchRecord(matrix_name, kind, (group_size if group_size is not None else 32)
                       if kind == "rgcsr" else None, "double" if prec == F64 else "single",
                       o.repetitions, m.nnz, med, measured_gflops(m.nnz, med),
                       fill.fill_percent, fill.artificial_zeros,
                       fill.bytes_double if prec == F64 else fill.bytes_single, checksum)
