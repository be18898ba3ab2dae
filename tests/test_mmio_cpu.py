"""Matrix Market ingestion (csrc/gen/mmio.cpp) against the
reference's own read_matrix_market / write_matrix_market compiled in place
(oracle/_ref): identical structure for every header kind, identical error
messages (with line numbers) for malformed files."""
import numpy as np
import pytest

from paper_2207_13848_b200 import gen
from tests.util import digest

pytestmark = pytest.mark.skipif(not __import__("oracle.pyoracle", fromlist=["Reference"]).Reference.available(),
                                reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def ref():
    from oracle.pyoracle import Reference
    return Reference()


def same(m, r):
    rows, cols, rpt, col = r
    return (m.rows, m.cols) == (rows, cols) and digest(m.rpt) == digest(rpt) and digest(m.col) == digest(col)


def entries_text(rng, n, rows, cols, nvals, diag_only_upper=False):
    lines = []
    for _ in range(n):
        i, j = int(rng.integers(1, rows + 1)), int(rng.integers(1, cols + 1))
        if diag_only_upper and i < j:
            i, j = j, i
        vals = " ".join(f"{rng.normal():.6g}" for _ in range(nvals))
        lines.append(f"{i} {j} {vals}".rstrip())
    return lines


KINDS = [("pattern", "general", 0), ("real", "general", 1), ("integer", "symmetric", 1),
         ("complex", "hermitian", 2), ("real", "skew-symmetric", 1), ("pattern", "symmetric", 0)]


@pytest.mark.parametrize("field,sym,nv", KINDS)
def test_read_matches_reference(ref, tmp_path, field, sym, nv):
    rng = np.random.default_rng(hash((field, sym)) % 2**32)
    rows, cols = (300, 300) if sym != "general" else (250, 400)
    body = entries_text(rng, 3000, rows, cols, nv, diag_only_upper=sym != "general")
    body += body[:40]  # duplicates
    n = len(body)
    # comments and blank lines between entries
    body.insert(5, "% a comment")
    body.insert(9, "")
    text = (f"%%MatrixMarket matrix coordinate {field.upper() if field == 'real' else field} {sym}\n"
            f"% generated\n\n{rows} {cols} {n}\n" + "\n".join(body) + "\n")
    p = tmp_path / "m.mtx"
    p.write_text(text)
    m = gen.read_matrix_market(p, threads=4)
    assert same(m, ref.read_matrix_market(p))


def test_write_round_trip(ref, tmp_path):
    a = gen.synthetic("power-law", 3000, 2500, 9.0, 4, 0, 0.8)
    p, q = tmp_path / "ours.mtx", tmp_path / "ref.mtx"
    gen.write_matrix_market(p, a)
    ref.write_matrix_market(q, a)
    assert p.read_bytes() == q.read_bytes()
    assert same(gen.read_matrix_market(p), (a.rows, a.cols, a.rpt, a.col))


BAD = {
    "header": "%%MatrixMarket matrix coordinate real\n2 2 1\n1 1 1\n",
    "object": "%%MatrixMarket vector coordinate real general\n2 2 1\n1 1 1\n",
    "format": "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n",
    "field": "%%MatrixMarket matrix coordinate quaternion general\n2 2 1\n1 1 1\n",
    "symmetry": "%%MatrixMarket matrix coordinate real upper\n2 2 1\n1 1 1\n",
    "nosize": "%%MatrixMarket matrix coordinate real general\n% only comments\n\n",
    "negative": "%%MatrixMarket matrix coordinate real general\n2 -2 1\n1 1 1\n",
    "truncated": "%%MatrixMarket matrix coordinate real general\n3 3 4\n1 1 1\n2 2 1\n% c\n3 3 1\n",
    "outside": "%%MatrixMarket matrix coordinate pattern general\n3 3 2\n1 1\n4 1\n",
    "trailing": "%%MatrixMarket matrix coordinate pattern general\n3 3 2\n1 1\n2 2 7\n",
    "notint": "%%MatrixMarket matrix coordinate pattern general\n3 3 1\nx 1\n",
    "noval": "%%MatrixMarket matrix coordinate real general\n3 3 2\n1 1 abc\n2 2 1\n",
    "sizetrail": "%%MatrixMarket matrix coordinate real general\n3 3 1 9\n1 1 1\n",
}


@pytest.mark.parametrize("kind", sorted(BAD))
def test_parse_errors_match_reference(ref, tmp_path, kind):
    p = tmp_path / f"{kind}.mtx"
    p.write_text(BAD[kind])
    with pytest.raises(RuntimeError) as r_err:
        ref.read_matrix_market(p)
    with pytest.raises(gen.ParseError) as o_err:
        gen.read_matrix_market(p)
    assert str(o_err.value) == str(r_err.value)


def test_missing_value_consumes_next_line_like_reference(ref, tmp_path):
    # strtod skips the newline: a value missing at the end of a line is read
    # from the next line, exactly as in the reference
    p = tmp_path / "quirk.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real general\n3 3 2\n1 1\n2 2\n3 3 5\n")
    try:
        r = ref.read_matrix_market(p)
    except RuntimeError as e:
        with pytest.raises(gen.ParseError) as o:
            gen.read_matrix_market(p)
        assert str(o.value) == str(e)
        return
    assert same(gen.read_matrix_market(p), r)
