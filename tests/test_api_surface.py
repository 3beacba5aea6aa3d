"""The drop-in package exports the reference's public names with the
reference's call signatures; the contract was recorded from
the reference by tests/golden/make_api_surface.py."""
import inspect
import json
import os

import pytest

import paper_1910_02371_b200 as cp

SURFACE = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "api_surface.json")))
# the sklearn-style estimator is outside the hot-path scope
OUT_OF_SCOPE = {"CPCompletion"}


def test_every_reference_name_is_exported():
    missing = [n for n in SURFACE["all"] if n not in OUT_OF_SCOPE and not hasattr(cp, n)]
    assert missing == []
    assert set(SURFACE["all"]) - OUT_OF_SCOPE <= set(cp.__all__)


@pytest.mark.parametrize("name", sorted(SURFACE["signatures"]))
def test_signature_matches_reference(name):
    want = SURFACE["signatures"][name]
    got = list(inspect.signature(getattr(cp, name)).parameters.values())
    # the reference's parameters, in order, with the same kinds and defaults;
    # extra trailing keyword parameters (device-side options) are allowed if
    # they have defaults
    assert len(got) >= len(want), name
    for p, (pname, kind, default) in zip(got, want):
        assert p.name == pname, (name, p.name, pname)
        assert p.kind.name == kind, (name, pname)
        have = None if p.default is inspect.Parameter.empty else repr(p.default)
        assert have == default, (name, pname, have, default)
    for p in got[len(want):]:
        assert p.default is not inspect.Parameter.empty, (name, p.name)
