"""The 2m+1 / last-m interleaved benchmark protocol (reference
autoselect.py:90-115) with a scripted clock, as the reference's own tests
inject timings (tests/test_autoselect.py:9-27)."""

import os

import pytest

from paper_2501_14490_b200 import protocol


class ScriptedTimer:
    def __init__(self, script):
        self.script = {k: list(v) for k, v in script.items()}
        self.calls = []

    def __call__(self, fn):
        name = fn()
        self.calls.append(name)
        return self.script[name].pop(0)


def test_last_m_of_2m_plus_1():
    t = ScriptedTimer({"a": [100.0, 50.0, 9.0, 1.0, 2.0]})
    assert protocol.benchmark_candidate(lambda: "a", m=2, timer=t) == 1.5
    assert len(t.calls) == 5
    with pytest.raises(ValueError):
        protocol.benchmark_candidate(lambda: "a", m=0, timer=t)


def test_interleaved_round_robin_and_best():
    t = ScriptedTimer({"x": [9, 9, 9, 3, 5], "y": [1, 1, 1, 4, 4]})
    rep = protocol.benchmark_interleaved({"x": lambda: "x", "y": lambda: "y"}, m=2, timer=t)
    assert t.calls == ["x", "y"] * 5  # interleaved, not one candidate after the other
    assert rep.as_dict() == {"x": 4.0, "y": 4.0}
    t = ScriptedTimer({"x": [9, 9, 9, 3, 5], "y": [1, 1, 1, 4, 3]})
    rep = protocol.benchmark_interleaved({"x": lambda: "x", "y": lambda: "y"}, m=2, timer=t)
    assert rep.best.name == "y" and "best=y" in rep.to_text()


def test_plan_env_restores_knobs():
    os.environ.pop("PSN_TEAMS_FWD", None)
    seen = []
    run = protocol.plan_variant(lambda: seen.append(os.environ.get("PSN_TEAMS_FWD")), PSN_TEAMS_FWD=4)
    run()
    assert seen == ["4"] and "PSN_TEAMS_FWD" not in os.environ
