"""Matrix Market ingest against the reference parser
(src/matrix_market.cpp:61-138, tests/test_matrix_core.cpp:126-252).

CPU: every rejection carries the reference's line number and message (the
parse fails before anything touches the GPU).  GPU: accepted files give the
reference's canonical matrix bitwise (duplicates summed in its order)."""
import numpy as np
import pytest
import torch

import oracle as orc
from helpers import bitwise
from paper_1012_2270_b200 import spmvkit as sk

BAD = [  # (text, line) — tests/test_matrix_core.cpp:196-216 plus count / shape errors
    ("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n", 1),
    ("%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1\n", 1),
    ("%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 1\n2 1 1\n", 1),
    ("%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n", 1),
    ("%%MatrixMarket vector coordinate real general\n1 1 1\n1 1 1\n", 1),
    ("not a banner\n", 1),
    ("", 1),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n", 3),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n", 3),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n", 3),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\n2 2 1.0\n", 4),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 3 1\n1 1 1.0\n", 2),
    ("%%MatrixMarket matrix coordinate real general\n% only comments\n", 3),
    ("%%MatrixMarket matrix coordinate real general\n2 x 1\n", 2),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0 junk\n", 3),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n\n% c\n1 q 1.0\n", 5),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\nbad line\n", 4),
]


@pytest.mark.parametrize("text,line", BAD)
def test_rejections_carry_reference_line_numbers(text, line):
    with pytest.raises(sk.MatrixMarketError) as e:
        sk.parse_matrix_market(text)
    assert e.value.line == line
    assert str(e.value).startswith(f"line {line}: ")
    if orc.ref_available():
        m, rline, rmsg = orc.RefMatrix.mm_parse(text.encode())
        assert m is None and rline == line and rmsg == str(e.value)


def _big_bad(n, extra):
    """A large file (parsed in parallel chunks) with an error deep inside."""
    lines = ["%%MatrixMarket matrix coordinate real general", f"{n} {n} {n}"]
    lines += [f"{i + 1} {i + 1} {i}.5" for i in range(n)]
    if extra == "garbage":
        lines[2 + n // 2] = "7 x 1.0"
    else:
        lines.append("1 1 1.0")
    return "\n".join(lines) + "\n"


@pytest.mark.parametrize("extra", ["garbage", "too_many"])
def test_parallel_chunks_keep_first_error_line(extra):
    text = _big_bad(300_000, extra)
    with pytest.raises(sk.MatrixMarketError) as e:
        sk.parse_matrix_market(text, threads=8)
    want = 3 + 150_000 if extra == "garbage" else 3 + 300_000
    assert e.value.line == want
    if orc.ref_available():
        _, rline, rmsg = orc.RefMatrix.mm_parse(text.encode())
        assert rline == want and rmsg == str(e.value)


def _random_mm(seed, field="real", symmetry="general", dup=True):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 40))
    k = int(rng.integers(0, 3 * n))
    rows = rng.integers(1, n + 1, k)
    cols = rng.integers(1, n + 1, k)
    if symmetry == "symmetric":
        rows, cols = np.maximum(rows, cols), np.minimum(rows, cols)
    if not dup and k:
        keys = np.unique(rows * 1000 + cols)
        rows, cols = keys // 1000, keys % 1000
        k = len(rows)
    out = [f"%%MatrixMarket matrix coordinate {field} {symmetry}", "% generated", f"{n} {n} {k}"]
    for r, c in zip(rows, cols):
        if field == "pattern":
            out.append(f"{r} {c}")
        elif field == "integer":
            out.append(f"{r} {c} {int(rng.integers(-9, 10))}")
        else:
            out.append(f"{r} {c} {rng.standard_normal():.17g}")
    return "\r\n".join(out) + "\r\n" if seed % 5 == 0 else "\n".join(out) + "\n"


CASES = [(s, f, sym) for s in range(12) for f in ("real", "integer", "pattern")
         for sym in ("general", "symmetric")]


@pytest.mark.gpu
@pytest.mark.parametrize("seed,field,sym", CASES)
def test_accepted_files_match_reference(cuda, seed, field, sym):
    if not orc.ref_available():
        pytest.skip("oracle/_ref not built")
    text = _random_mm(seed, field, sym)
    ref, line, msg = orc.RefMatrix.mm_parse(text.encode())
    assert ref is not None, msg
    want = ref.to_csr()
    for prec in (8, 4):
        a = sk.parse_matrix_market(text, prec, threads=3)
        rp, col, val = a.to_host()
        assert bitwise(rp, want.rp) and bitwise(col, want.col)
        assert bitwise(val, want.val.astype(np.float64 if prec == 8 else np.float32))


@pytest.mark.gpu
def test_reference_examples_and_writer_round_trip(cuda, tmp_path):
    """tests/test_matrix_core.cpp:126-252 verbatim cases + write/load round trip."""
    a = sk.parse_matrix_market("%%MatrixMarket matrix coordinate real symmetric\n"
                               "2 2 2\n1 1 4.0\n2 1 3.0\n")
    rp, col, val = a.to_host()
    assert rp.tolist() == [0, 2, 3] and col.tolist() == [0, 1, 0] and val.tolist() == [4, 3, 3]
    a = sk.parse_matrix_market("%%MatrixMarket matrix coordinate integer general\n% a comment\n\n"
                               "2 2 1\n% another\n2 1 -3\n")
    assert a.to_host()[2].tolist() == [-3.0]
    a = sk.parse_matrix_market("%%MatrixMarket matrix coordinate real general\r\n1 1 1\r\n1 1 9.5\r\n")
    assert a.to_host()[2].tolist() == [9.5]
    if orc.ref_available():
        for seed in range(7, 17):
            r = orc.RefMatrix.random_small(seed, True, False)
            p = tmp_path / f"m{seed}.mtx"
            p.write_bytes(r.mm_write())
            rp, col, val = sk.load_matrix_market(str(p)).to_host()
            w = r.to_csr()
            assert bitwise(rp, w.rp) and bitwise(col, w.col) and bitwise(val, w.val)
    with pytest.raises(sk.MatrixMarketError) as e:
        p = tmp_path / "bad.mtx"
        p.write_text("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n")
        sk.load_matrix_market(str(p))
    assert e.value.line == 3 and str(e.value).startswith(str(p) + ": line 3: ")
    torch.cuda.synchronize()


@pytest.mark.gpu
@pytest.mark.skipif(not orc.ref_available(), reason="oracle/_ref not built")
def test_writer_matches_reference_bytes(cuda, tmp_path):
    """write_matrix_market / save_matrix_market (src/matrix_market.cpp:150-164):
    identical bytes to the reference writer, any thread count; parse round trip."""
    for seed in range(20, 40):
        r = orc.RefMatrix.random_small(seed, True, seed % 2 == 0)
        want = r.mm_write()
        w = r.to_csr()
        a = sk.build_csr(sk.TripletMatrix(w.rows, w.cols, w.rp, w.col, w.val))
        for threads in (1, 3, 0):
            assert sk.write_matrix_market(a, threads).encode() == want, (seed, threads)
        p = tmp_path / f"w{seed}.mtx"
        sk.save_matrix_market(p, a)
        assert p.read_bytes() == want
        rp, col, val = sk.load_matrix_market(p).to_host()
        assert bitwise(rp, w.rp) and bitwise(col, w.col) and bitwise(val, w.val)
    big = sk.CsrMatrix.stencil(7, 40)  # 64k rows: several formatting threads
    text = sk.write_matrix_market(big, 8)
    assert text == sk.write_matrix_market(big, 1)
    rp, col, val = sk.parse_matrix_market(text).to_host()
    rp2, col2, val2 = big.to_host()
    assert bitwise(rp, rp2) and bitwise(col, col2) and bitwise(val, val2)
    with pytest.raises(sk.SpmvkRuntimeError, match="for writing"):
        sk.save_matrix_market(tmp_path / "no" / "such" / "dir.mtx", big)


@pytest.mark.gpu
def test_matrix_stats(cuda):
    """matrix_stats (src/triplet.cpp:57-69)."""
    m = sk.canonicalize([(0, 0, 1.0), (0, 2, 2.0), (2, 1, 3.0)], 4, 5)
    s = sk.matrix_stats(m)
    assert (s.num_rows, s.nnz, s.row_len_max, s.row_len_min) == (4, 3, 2, 0)
    assert s.row_len_mean == 0.75 and s.density_percent == 100.0 * 3 / 20
    with pytest.raises(sk.InvalidArgument, match="matrix has zero rows"):
        sk.matrix_stats(sk.canonicalize([], 0, 3))
