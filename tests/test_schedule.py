"""The product's host-side DTS schedule against the oracle's reading of the paper
(P:535 endpoints, P:708 decay window / Top-1 switch) and the C5 workload definition."""
import math

from harness import configs
from oracle import dts_moe as O
from paper_2112_14397_b200.schedule import DTSSchedule, c5_sweep


def test_schedule_matches_oracle_and_paper_endpoints():
    s = DTSSchedule()
    assert s.tau(0) == 2.0 and s.tau(15000) == 0.3 and s.tau(10 ** 6) == 0.3
    for it in (0, 1, 777, 7500, 14999, 15000, 20000):
        assert abs(s.tau(it) - O.temperature_at(it)) < 1e-12
        assert abs(DTSSchedule(shape="exp").tau(it) - O.temperature_at(it, shape="exp")) < 1e-12
    assert not s.top1(14999) and s.top1(15000)
    assert s.at(3) == (s.tau(3), 0.001, False)


def test_c5_sweep_equals_workload_config():
    got = list(c5_sweep())
    assert len(got) == 20
    for (t, c), (t2, c2) in zip(got, configs.C5.schedule):
        assert abs(t - t2) < 1e-15 and abs(c - c2) < 1e-15
    assert abs(got[-1][0] - 0.05) < 1e-15 and math.isclose(got[0][0], 2.0)
