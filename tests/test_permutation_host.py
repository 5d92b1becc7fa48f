"""Host-side Permutation / parse_permutation (src/reorder.cpp:12-33, 63-91;
tests/test_reorder.cpp:55-60, 161-172) -- no GPU needed."""
import pytest

from paper_1012_2270_b200 import spmvkit as sk


def test_bijections_and_identity():
    assert sk.Permutation([1, 0, 2]).map().tolist() == [1, 0, 2]
    for bad in ([0, 0], [2, 0], [-1, 0]):
        with pytest.raises(sk.InvalidArgument, match="not a bijection"):
            sk.Permutation(bad)
    assert sk.Permutation.identity(3).map().tolist() == [0, 1, 2]
    assert sk.Permutation([2, 0, 1]).inverse().tolist() == [1, 2, 0]
    assert sk.Permutation([]).size() == 0


def test_parse_permutation(tmp_path):
    assert sk.parse_permutation("1\n0\n").map().tolist() == [1, 0]
    assert sk.parse_permutation("2\n0\n1\n").map().tolist() == [2, 0, 1]
    assert sk.parse_permutation("  1\r\n\n\t0 \n").map().tolist() == [1, 0]
    for bad, msg in (("0\n0\n", "not a bijection"), ("2\n0\n", "not a bijection"),
                     ("a\nb\n", "line 1: expected an index, got 'a'"),
                     ("-1\n0\n", "line 1: expected a single 0-based index, got '-1'"),
                     ("0\n1 2\n", "line 2: expected a single 0-based index")):
        with pytest.raises(sk.InvalidArgument, match=msg):
            sk.parse_permutation(bad)
    p = tmp_path / "p.txt"
    p.write_text("1\n2\n0\n")
    assert sk.load_permutation(p).map().tolist() == [1, 2, 0]
    with pytest.raises(sk.SpmvkRuntimeError, match="cannot open"):
        sk.load_permutation(tmp_path / "missing.txt")
