"""The input side of the path: the library's load_dataset /
save_dataset / split / enlarge (csrc/dataset.cuh) against the oracle
restatement (oracle/lane_oracle.c) and, where it was built here, the
unmodified reference (oracle/_ref, proj/src/dataset.cpp).  Host-only code:
these run on CPU."""
import os

import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2001_04206_b200 import lane

IRIS = os.path.join(os.path.dirname(__file__), "golden", "iris_normalized.txt")
needs_ref = pytest.mark.skipif(not po.ref_available(), reason="oracle/_ref not built")


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def assert_bitwise(a, b):
    np.testing.assert_array_equal(bits(a), bits(b))


def test_load_iris_matches_oracle():
    d = lane.load_dataset(IRIS, 4, 3)
    X, T = po.load_dataset(IRIS, 4, 3)
    assert d.size() == 150 and d.feature_width == 4 and d.class_count == 3
    assert_bitwise(d.features, X)
    assert_bitwise(d.labels, T)


@pytest.mark.parametrize("frac,seed", [(0.9, 42), (0.5, 1), (0.01, 7), (0.999, 3)])
def test_split_matches_oracle(frac, seed):
    d = lane.load_dataset(IRIS, 4, 3)
    a, b = lane.split(d, frac, seed)
    Xa, Ta, Xb, Tb = po.split(d.features, d.labels, frac, seed)
    assert a.size() == len(Xa) and b.size() == len(Xb)
    assert_bitwise(a.features, Xa)
    assert_bitwise(a.labels, Ta)
    assert_bitwise(b.features, Xb)
    assert_bitwise(b.labels, Tb)


def test_split_of_plain_arrays():
    X, T = po.synthetic_dataset(5, 2, 33, 4)
    a, b = lane.split(lane.DataSet(X, T), 0.7, 11)
    Xa, Ta, Xb, Tb = po.split(X, T, 0.7, 11)
    assert_bitwise(a.features, Xa)
    assert_bitwise(b.labels, Tb)


@pytest.mark.parametrize("frac", [0.0, 1.0, -0.5, 1.5, float("nan")])
def test_split_rejects_fraction(frac):
    d = lane.load_dataset(IRIS, 4, 3)
    with pytest.raises(lane.ConfigError):
        lane.split(d, frac, 1)


def _oracle_enlarge(X, T, factor, noise, rng):
    n, F = X.shape
    C_ = T.shape[1]
    Xo = np.zeros((n * factor, F), np.float32)
    To = np.zeros((n * factor, C_), np.float32)
    po.oracle_lib().lo_enlarge(np.ascontiguousarray(X).reshape(-1), np.ascontiguousarray(T).reshape(-1), n, F,
                               C_, factor, noise, rng, Xo.reshape(-1), To.reshape(-1))
    return Xo, To


@pytest.mark.parametrize("factor,noise", [(1, 0.0), (3, 0.0), (2, 0.05), (4, 0.5)])
def test_enlarge_matches_oracle(factor, noise):
    import ctypes as C
    d = lane.load_dataset(IRIS, 4, 3)
    rng = lane.SeededRng(42)
    orng = (C.c_uint64 * 2)()
    po.oracle_lib().lo_rng_init(C.cast(orng, C.c_void_p), 42)
    for _ in range(2):  # the generator carries over between calls
        e = lane.enlarge(d, factor, noise, rng)
        Xo, To = _oracle_enlarge(d.features, d.labels, factor, noise, C.cast(orng, C.c_void_p))
        assert e.size() == 150 * factor
        assert_bitwise(e.features, Xo)
        assert_bitwise(e.labels, To)
        assert (e.features >= 0).all() and (e.features <= 1).all()


def test_enlarge_rejects_bad_arguments():
    d = lane.load_dataset(IRIS, 4, 3)
    with pytest.raises(lane.ConfigError):
        lane.enlarge(d, 0, 0.1, lane.SeededRng(1))
    with pytest.raises(lane.ConfigError):
        lane.enlarge(d, 2, -0.1, lane.SeededRng(1))


def test_save_load_round_trip(tmp_path):
    X, T = po.synthetic_dataset(7, 4, 50, 123)
    X[0, 0], X[1, 1] = 1e-30, 0.1  # denormal-ish and a non-representable decimal
    p = tmp_path / "ds.csv"
    lane.save_dataset(lane.DataSet(X, T), p)
    d = lane.load_dataset(p, 7, 4)
    assert_bitwise(d.features, X)
    assert_bitwise(d.labels, T)
    first = p.read_text().splitlines()[0].split(",")
    assert len(first) == 11 and first[0] == "%.9g" % float(X[0, 0])
    assert first[7:] == [("1" if v == 1 else "0") for v in T[0]]


# --------------------------------------------------------- parse rules ---
GOOD = "0.25,0.5,0.75,1,1,0,0\n"

CASES = {
    # name: (text, rows or the error class)
    "plain": (GOOD * 3, 3),
    "empty_lines": ("\n" + GOOD + "\n\n" + GOOD, 2),
    "crlf": (GOOD.replace("\n", "\r\n") * 2, 2),
    "no_final_newline": (GOOD + GOOD.strip(), 2),
    "trailing_comma": ("0.25,0.5,0.75,1,1,0,0,\n", 1),  # getline(',') adds no empty field
    "empty_file": ("", 0),
    "exponent": ("2.5e-1,5E-1,0.75,1,0,0,1\n", 1),
    "too_few": ("0.25,0.5,0.75,1,0\n", lane.ParseError),
    "too_many": ("0.25,0.5,0.75,1,1,0,0,0\n", lane.ParseError),
    "inner_empty": ("0.25,,0.75,1,1,0,0\n", lane.ParseError),
    "alpha": ("0.25,abc,0.75,1,1,0,0\n", lane.ParseError),
    "plus_sign": ("+0.25,0.5,0.75,1,1,0,0\n", lane.ParseError),  # from_chars rejects '+'
    "blank_in_field": ("0.25, 0.5,0.75,1,1,0,0\n", lane.ParseError),
    "trailing_junk": ("0.25x,0.5,0.75,1,1,0,0\n", lane.ParseError),
    "label_two": ("0.25,0.5,0.75,1,2,0,0\n", lane.ParseError),
    "label_half": ("0.25,0.5,0.75,1,0.5,0.5,0\n", lane.ParseError),
    "two_hot": ("0.25,0.5,0.75,1,1,1,0\n", lane.ParseError),
    "zero_hot": ("0.25,0.5,0.75,1,0,0,0\n", lane.ParseError),
    "bad_second_line": (GOOD + "1,2\n", lane.ParseError),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_parse_rules(tmp_path, name):
    text, want = CASES[name]
    p = tmp_path / f"{name}.csv"
    p.write_bytes(text.encode())
    if isinstance(want, int):
        d = lane.load_dataset(p, 4, 3)
        assert d.size() == want
        if want:
            assert d.labels.sum() == want
    else:
        with pytest.raises(want) as ei:
            lane.load_dataset(p, 4, 3)
        assert "line" in str(ei.value)


def test_parse_error_names_the_line(tmp_path):
    p = tmp_path / "bad.csv"
    p.write_text(GOOD + "\n" + GOOD + "0.1,0.2,0.3,0.4,0,2,0\n")
    with pytest.raises(lane.ParseError, match="line 4: label field must be 0 or 1"):
        lane.load_dataset(p, 4, 3)


def test_missing_file_is_io_error(tmp_path):
    with pytest.raises(lane.IoError, match="cannot open dataset file"):
        lane.load_dataset(tmp_path / "nope.csv", 4, 3)


@needs_ref
@pytest.mark.parametrize("name", sorted(CASES))
def test_parse_rules_match_reference(tmp_path, name):
    """Row count or failure identical to the reference's load_dataset."""
    text, _ = CASES[name]
    p = tmp_path / f"{name}.csv"
    p.write_bytes(text.encode())
    Xr = np.zeros((8, 4), np.float32)
    Tr = np.zeros((8, 3), np.float32)
    got = po.ref_lib().lr_load_dataset(str(p).encode(), 4, 3, Xr.reshape(-1), Tr.reshape(-1), 8)
    try:
        d = lane.load_dataset(p, 4, 3)
        mine = d.size()
    except lane.ParseError:
        mine = -1
    assert mine == got
    if got > 0:
        assert_bitwise(d.features, Xr[:got])
        assert_bitwise(d.labels, Tr[:got])


@needs_ref
def test_enlarge_matches_reference():
    d = lane.load_dataset(IRIS, 4, 3)
    Xr = np.zeros((450, 4), np.float32)
    Tr = np.zeros((450, 3), np.float32)
    assert po.ref_lib().lr_enlarge(d.features.reshape(-1), d.labels.reshape(-1), 150, 4, 3, 3, 0.05, 9,
                                   Xr.reshape(-1), Tr.reshape(-1)) == 0
    e = lane.enlarge(d, 3, 0.05, lane.SeededRng(9))
    assert_bitwise(e.features, Xr)
    assert_bitwise(e.labels, Tr)


@needs_ref
def test_parse_fuzz_matches_reference(tmp_path):
    """Random near-miss CSV files (mutated fields, separators, signs, blanks,
    line endings): the library's loader accepts exactly what the reference's
    load_dataset accepts, with bitwise equal rows."""
    rs = np.random.default_rng(20261017)
    atoms = ["0", "1", "0.5", "1e-3", "2.5E+1", "-0.25", ".5", "5.", "+1", " 1", "1 ", "", "nan", "inf",
             "-0", "1e", "0x1p-2", "1,0", "\t", "0.3333333333333333", "3.4028235e38", "1e-45", "abc"]
    for trial in range(400):
        lines = []
        for _ in range(int(rs.integers(1, 6))):
            feats = [str(np.float32(rs.uniform(0, 1))) for _ in range(4)]
            lab = ["0", "0", "0"]
            lab[int(rs.integers(3))] = "1"
            fields = feats + lab
            for _ in range(int(rs.integers(0, 3))):  # mutate a few fields
                fields[int(rs.integers(len(fields)))] = atoms[int(rs.integers(len(atoms)))]
            line = ",".join(fields)
            if rs.random() < 0.2:
                line += ","
            if rs.random() < 0.2:
                line += "\r"
            lines.append(line)
        if rs.random() < 0.3:
            lines.insert(int(rs.integers(len(lines) + 1)), "")
        p = tmp_path / f"fuzz{trial}.csv"
        p.write_bytes(("\n".join(lines) + ("\n" if rs.random() < 0.5 else "")).encode())
        Xr = np.zeros((16, 4), np.float32)
        Tr = np.zeros((16, 3), np.float32)
        got = po.ref_lib().lr_load_dataset(str(p).encode(), 4, 3, Xr.reshape(-1), Tr.reshape(-1), 16)
        try:
            d = lane.load_dataset(p, 4, 3)
            mine = d.size()
        except lane.ParseError:
            mine = -1
        assert mine == got, (trial, p.read_text())
        if got > 0:
            assert_bitwise(d.features, Xr[:got])
            assert_bitwise(d.labels, Tr[:got])
