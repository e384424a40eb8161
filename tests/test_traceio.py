"""EXFLOW-TRACE v1 I/O (paper_2401_08383_b200/traceio.py) against the
reference's parse cases (proj/tests/test_trace.cpp:46-92) and its fixture
proj/data/two_token_demo.trace (committed copy under tests/golden/)."""
import os

import numpy as np
import pytest

from paper_2401_08383_b200 import traceio as tio

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_minimal_well_formed():  # test_trace.cpp:46-54
    paths, E = tio.parse_trace("EXFLOW-TRACE v1\nE 2 L 2\n0 0\n1 1\n")
    assert E == 2 and paths.tolist() == [[0, 0], [1, 1]] and paths.dtype == np.int32


def test_out_of_range_id_reports_line():  # :56-60
    with pytest.raises(tio.ParseError, match=r"expert id 2 out of range \[0,2\) at line 4"):
        tio.parse_trace("EXFLOW-TRACE v1\nE 2 L 2\n0 0\n0 2\n")


def test_short_path():  # :62-65
    with pytest.raises(tio.ParseError, match="path length 1 != L=2"):
        tio.parse_trace("EXFLOW-TRACE v1\nE 2 L 2\n0\n")


def test_comments_and_blank_lines():  # :67-72
    paths, E = tio.parse_trace("# preamble\nEXFLOW-TRACE v1\n# dims\nE 3 L 2\n\n0 2\n# done\n1 1\n")
    assert E == 3 and paths.tolist() == [[0, 2], [1, 1]]


@pytest.mark.parametrize("text,msg", [
    ("bogus\n", "missing or unsupported EXFLOW-TRACE header at line 1"),
    ("EXFLOW-TRACE v1\nE 0 L 2\n", "E must be >= 1"),
    ("EXFLOW-TRACE v1\nE 2 L 1\n0\n", "L must be >= 2"),
    ("EXFLOW-TRACE v1\nE 2 L 2\n", "no token paths"),
    ("EXFLOW-TRACE v1\nE 2 L 2\n0 x\n", "invalid token 'x' at line 3"),
    ("EXFLOW-TRACE v1\nE 2 L 2\n0 +1\n", "invalid token '\\+1' at line 3"),  # from_chars: no '+'
    ("", "missing or unsupported EXFLOW-TRACE header at line 1"),
    ("EXFLOW-TRACE v1\n", "missing 'E <experts> L <layers>' line"),
    ("EXFLOW-TRACE v1\nE 2 X 2\n", "expected 'E <experts> L <layers>' at line 2"),
])
def test_header_and_dimension_errors(text, msg):  # :74-84
    with pytest.raises(tio.ParseError, match=msg):
        tio.parse_trace(text)


def test_crlf_and_round_trip(tmp_path):  # :86-92
    rng = np.random.default_rng(3)
    paths = rng.integers(0, 8, size=(50, 4)).astype(np.int32)
    text = tio.serialize_trace(paths, 8)
    assert text.startswith("EXFLOW-TRACE v1\nE 8 L 4\n")
    back, E = tio.parse_trace(text.replace("\n", "\r\n"))
    assert E == 8 and np.array_equal(back, paths)
    f = tmp_path / "t.trace"
    tio.save_trace(f, paths, 8)
    back, _ = tio.load_trace(f)
    assert np.array_equal(back, paths)


def test_reference_fixture():
    paths, E = tio.load_trace(os.path.join(GOLDEN, "two_token_demo.trace"))
    assert E == 8 and paths.tolist() == [[0, 4, 2], [5, 5, 4]]


def test_validate_messages():  # RoutingTrace::validate, trace.cpp:48-70
    with pytest.raises(ValueError, match=r"expert id out of range \[0,4\)"):
        tio.serialize_trace(np.array([[0, 4]]), 4)
    with pytest.raises(ValueError, match="num_layers must be >= 2"):
        tio.serialize_trace(np.array([[0], [1]]), 4)
    with pytest.raises(RuntimeError, match="cannot open trace file"):
        tio.load_trace("/nonexistent/dir/t.trace")
