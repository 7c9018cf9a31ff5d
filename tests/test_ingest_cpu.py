"""Host ingestion of the reference CLI's text format (cli.py:60-70): the
native parser (libpmh.so, no device work) against the reference's own
parse of a fixture text (tests/golden/ingest.npz) and against the exact
Python restatement on randomised texts, valid and invalid."""
import numpy as np
import pytest

from golden_io import load
from paper_1911_00675_b200 import _lib
from paper_1911_00675_b200.errors import EmptyInputError, InvalidParamsError
from paper_1911_00675_b200.ingest import (_python_path, parse_weighted_text, read_sets_csr,
                                          read_weighted_lines, format_signature)


def test_reference_fixture():
    z = load("ingest")
    text = str(z["text"])
    ids, w = parse_weighted_text(text)
    assert np.array_equal(ids, z["ids"])
    np.testing.assert_array_equal(w, z["weights"])   # inf / nan / -2.5 included
    # the fixture is entirely within the native grammar
    cap = text.count("\n") + 1
    a, b = np.empty(cap, np.uint64), np.empty(cap, np.float64)
    assert _lib.load().pmh_parse_weighted_text(text.encode(), len(text), a.ctypes.data,
                                               b.ctypes.data, cap) == ids.size


def _rand_int_token(rng):
    v = int(rng.integers(0, 2**63)) * int(rng.integers(1, 3))
    kind = rng.integers(0, 4)
    if kind == 0:
        s = str(v)
    elif kind == 1:
        s = ("0x" if rng.random() < 0.5 else "0X") + format(v, "x" if rng.random() < 0.5 else "X")
    elif kind == 2:
        s = "0o" + format(v, "o")
    else:
        s = "0b" + format(v, "b")
    if rng.random() < 0.2 and len(s) > 3:      # an underscore between two digits
        i = int(rng.integers(3, len(s)))
        if s[i - 1].isalnum() and s[i].isalnum() and s[i - 1] not in "xXoObB":
            s = s[:i] + "_" + s[i:]
    if rng.random() < 0.1:
        s = "+" + s
    return s


def _rand_float_token(rng):
    x = float(rng.exponential()) * 10.0 ** int(rng.integers(-5, 6))
    kind = rng.integers(0, 5)
    return [repr(x), f"{x:e}", f"{x:.3f}", "inf" if rng.random() < 0.5 else "1_0.5", "7"][kind]


BAD = ["-5", "007", "0x", "1__0", "_1", "1_", "0x1g", "1.5", "abc", "0b102"]
BAD_W = ["1__0", "0x1p3", "nan(1)", "1e", "--1", "_5", "5_"]


@pytest.mark.parametrize("seed", range(40))
def test_native_equals_restatement(seed):
    rng = np.random.default_rng(seed)
    lines = []
    for _ in range(int(rng.integers(1, 60))):
        r = rng.random()
        if r < 0.08:
            lines.append("# comment " + str(rng.integers(100)))
        elif r < 0.14:
            lines.append("   " if rng.random() < 0.5 else "")
        else:
            tok = [_rand_int_token(rng)]
            if rng.random() < 0.8:
                tok.append(_rand_float_token(rng))
            if rng.random() < 0.1:
                tok.append("extra")
            sep = "\t" if rng.random() < 0.2 else " " * int(rng.integers(1, 3))
            lines.append(" " * int(rng.integers(0, 2)) + sep.join(tok))
    if seed % 4 == 3:                           # one malformed line
        lines.insert(int(rng.integers(0, len(lines) + 1)),
                     (BAD[seed % len(BAD)] + " 1") if seed % 8 == 3 else ("5 " + BAD_W[seed % len(BAD_W)]))
    text = "\n".join(lines) + ("\n" if seed % 2 else "")
    try:
        exp = _python_path(text.encode())
    except (ValueError, OverflowError) as err:
        with pytest.raises(type(err)):
            parse_weighted_text(text)
        return
    got = parse_weighted_text(text)
    assert np.array_equal(got[0], exp[0])
    np.testing.assert_array_equal(got[1], exp[1])


def test_bare_cr_and_crlf():
    a = parse_weighted_text("1 2\r\n3 4\r\n")
    assert a[0].tolist() == [1, 3] and a[1].tolist() == [2.0, 4.0]
    b = parse_weighted_text("1 2\r3 4")           # bare CR: the reference splits here
    assert b[0].tolist() == [1, 3]


def test_read_sets_csr_and_validation(tmp_path):
    p = tmp_path / "a.txt"
    p.write_text("1 0.5\n2 1.5\n")
    batch = read_sets_csr([str(p), b"7 2\n8\n9 3\n"])
    assert batch.offsets.tolist() == [0, 2, 5]
    assert batch.ids.tolist() == [1, 2, 7, 8, 9]
    with pytest.raises(InvalidParamsError):
        read_sets_csr([b"1 1\n1 2\n"])
    with pytest.raises(InvalidParamsError):
        read_sets_csr([b"1 0\n"])
    with pytest.raises(EmptyInputError):
        read_sets_csr([b"# nothing\n"])
    assert read_weighted_lines(["0x10 2", "", "#"]) == [(16, 2.0)]
    assert format_signature(np.array([3, 1], np.uint64)) == "3\n1\n"
