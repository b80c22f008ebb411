"""Problem files (grid_problem.py:431-529): documents written by the reference's
save_problem load into the same dense arrays the golden cases hold, and our writer emits
the reference's document byte-for-byte in content (dict equality after a round trip)."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR, load_golden

CASES = ["boundary", "time_varying"]


@pytest.mark.parametrize("name", CASES)
def test_reference_json_loads_to_golden_arrays(name):
    from paper_2304_04980_b200 import arrays_from_problem, load_problem

    ga_ref, rec = load_golden(name)
    prob = load_problem(os.path.join(GOLDEN_DIR, f"{name}_problem.json"))
    ga = arrays_from_problem(prob)
    for key in ("A", "B", "R", "C", "Q", "dyn_class", "cost_class", "offset"):
        assert np.array_equal(getattr(ga, key), getattr(ga_ref, key)), key
    assert np.array_equal(ga.offset, rec["ref_offset"])


@pytest.mark.parametrize("name", CASES)
def test_roundtrip_matches_reference_document(name, tmp_path):
    from paper_2304_04980_b200 import load_problem, problem_to_dict, save_problem

    path = os.path.join(GOLDEN_DIR, f"{name}_problem.json")
    with open(path) as fh:
        ref_doc = json.load(fh)
    prob = load_problem(path)
    assert problem_to_dict(prob) == ref_doc
    out = tmp_path / "p.json"
    save_problem(prob, out)
    with open(out) as fh:
        assert json.load(fh) == ref_doc


def test_rejects_foreign_document():
    from paper_2304_04980_b200 import problem_from_dict

    with pytest.raises(ValueError, match="grid-lq-problem"):
        problem_from_dict({"format": "something-else"})
