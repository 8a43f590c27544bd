"""lp2d v1 text instances (io.hpp), the reference's replay format. CPU only.
Golden strings from proj/tests/test_generate.cpp:150-185."""
import numpy as np
import pytest


def test_round_trip_bit_exact(P):
    from paper_1902_04995_b200.lp2d import problem_from_text, to_text

    p = P.gen(50, 31337, P.GenKind.feasible_random, 0.125)
    text = to_text(p)
    q = problem_from_text(text)
    assert np.array_equal(q.constraints, p.constraints) and q.c == p.c and q.bound_m == p.bound_m
    assert to_text(q) == text


def test_golden_format(P):
    from paper_1902_04995_b200.lp2d import to_text

    p = P.Problem((1.0, 0.5), [[-0.25, 1.0, 3.5]])
    assert to_text(p) == ("lp2d v1 m=1 M=1.0000000000000000e+07\n"
                          "c 1.0000000000000000e+00 5.0000000000000000e-01\n"
                          "h -2.5000000000000000e-01 1.0000000000000000e+00 "
                          "3.5000000000000000e+00\n")


@pytest.mark.parametrize("text", [
    "nonsense",
    "lp2d v2 m=0 M=1.0\nc 1 0\n",
    "lp2d v1 m=1 M=1.0\nc 1 0\n",          # missing constraint line
    "lp2d v1 m=1 M=1.0\nc 1 0\nh 0 0 1\n",  # zero normal
    "lp2d v1 m=1 M=-2.0\nc 1 0\nh 1 0 1\n",  # negative box
])
def test_malformed_rejected(P, text):
    from paper_1902_04995_b200.lp2d import ParseError, problem_from_text

    with pytest.raises(ParseError):
        problem_from_text(text)
