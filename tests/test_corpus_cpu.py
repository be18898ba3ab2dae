"""Synthetic corpus generator (SURVEY §8f-3 input side) against the
reference's own generate_synthetic / synthetic_name compiled in place
(oracle/_ref): identical matrices and names, including the default corpus."""
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


SPECS = gen.DEFAULT_CORPUS + [
    (1000, 1000, "uniform", 4.0, 7, 0, 1.0),
    (5000, 5000, "banded", 10.0, 1, 64, 1.0),
    (3000, 4000, "banded", 7.5, 9, 0, 1.0),      # default bandwidth
    (8000, 8000, "power-law", 12.0, 3, 0, 0.8),
    (500, 40, "uniform", 40.0, 5, 0, 1.0),       # target == cols
    (0, 10, "uniform", 1.0, 5, 0, 1.0),
    (10, 0, "uniform", 0.0, 5, 0, 1.0),
]


@pytest.mark.parametrize("spec", SPECS, ids=lambda s: f"{s[2]}-{s[0]}x{s[1]}-{s[3]}-{s[4]}")
def test_synthetic_matches_reference(ref, spec):
    rows, cols, model, target, seed, bw, skew = spec
    m = gen.synthetic(model, rows, cols, target, seed, bw, skew)
    r, c, rpt, col, name = ref.generate_synthetic(model, rows, cols, target, seed, bw, skew)
    assert (m.rows, m.cols) == (r, c)
    assert digest(m.rpt) == digest(rpt) and digest(m.col) == digest(col)
    assert gen.synthetic_name(model, rows, cols, target, seed, bw, skew) == name
    assert gen.parse_synthetic_spec(name) == dict(model=model, rows=rows, cols=cols, target=target,
                                                  seed=seed, bandwidth=bw if model == "banded" else 0,
                                                  skew=skew if model == "power-law" else 1.0)


def test_synthetic_rejects_infeasible(ref):
    with pytest.raises(ValueError):
        gen.synthetic("uniform", 10, 5, 6.0, 1)
    with pytest.raises(ValueError):
        ref.generate_synthetic("uniform", 10, 5, 6.0, 1)
    with pytest.raises(ValueError):
        gen.parse_synthetic_spec("synth:cubic:3x3")
    with pytest.raises(ValueError):
        gen.parse_synthetic_spec("synth:uniform:3by3")
