"""CPU: host logic of the f3 harness backend (paper_2510_18413_b200/harness.py)
— labels, validation, needle reports, emitters and the JSON library's number
formatting — against the reference (oracle/_ref) where it is built and against
literals from the reference's own tests."""
import numpy as np
import pytest

from paper_2510_18413_b200 import harness as H
from paper_2510_18413_b200._lib import ConfigError


def test_labels():  # sweep.hpp:27-30 examples, sweep.cpp:146-161
    assert H.PolicySpec("adamas").label() == "adamas-2bit-l1"
    assert H.PolicySpec("adamas", with_hadamard=False).label() == "adamas-2bit-l1-nohadamard"
    assert H.PolicySpec("adamas", bits=3, metric="euclidean_sq").label() == "adamas-3bit-l2"
    assert H.PolicySpec("window", sink=4).label() == "window-sink4"
    assert H.PolicySpec("quest", page_size=16).label() == "quest-p16"
    assert H.PolicySpec("oracle").label() == "oracle"


def test_validation():
    with pytest.raises(ConfigError, match="at least one budget"):
        H.SweepConfig([], [H.PolicySpec()]).validate()
    with pytest.raises(ConfigError, match="positive"):
        H.SweepConfig([0], [H.PolicySpec()]).validate()
    with pytest.raises(ConfigError, match="ascending"):
        H.SweepConfig([16, 16], [H.PolicySpec()]).validate()
    with pytest.raises(ConfigError, match="at least one policy"):
        H.SweepConfig([16], []).validate()
    with pytest.raises(ConfigError, match="bits"):
        H.SweepConfig([16], [H.PolicySpec(bits=4)]).validate()
    with pytest.raises(ConfigError, match="page_size"):
        H.SweepConfig([16], [H.PolicySpec("quest", page_size=0)]).validate()
    with pytest.raises(ConfigError, match="power of two"):
        H.WorkloadSpec(head_dim=48).validate()
    with pytest.raises(ConfigError, match="needle position"):
        H.WorkloadSpec(seq_len=8, distribution="planted_needle", position=8).validate()
    H.WorkloadSpec(seq_len=8, head_dim=32).validate()


def test_format_number_literals():
    cases = [(1.0, "1.0"), (0.5, "0.5"), (0.0, "0.0"), (-0.0, "-0.0"), (1e-05, "1e-05"), (0.0001, "0.0001"),
             (1e15, "1e+15"), (123456789012345.0, "123456789012345.0"), (100.0, "100.0"), (1.5e300, "1.5e+300"),
             (5e-324, "5e-324"), (float("nan"), "null"), (0.2755905511811024, "0.27559055118110237")]
    for v, s in cases:
        assert H.format_number(v) == s, v


def test_cached_powers_table():
    # first / middle / last entries of the JSON library's table (json.hpp 3.11.3)
    assert H._CACHED[0] == (0xAB70FE17C79AC6CA, -1060, -300)
    assert H._CACHED[38] == (0x9C40000000000000, -50, 4)
    assert H._CACHED[-1] == (0x9E19DB92B4E31BA9, 1013, 324)


def test_format_number_vs_reference(reference):
    rng = np.random.default_rng(7)
    vals = [j / k for k in range(1, 120) for j in range(k + 1)]
    vals += list(rng.random(20000)) + list(10 ** rng.uniform(-300, 300, 20000)) + list(-rng.random(100))
    vals = np.array(vals)
    lines = reference.rows_to_csv(vals).splitlines()[1:]
    got = [H.format_number(v) for v in vals]
    assert [ln.split(",")[3] for ln in lines] == got


def _rows():
    rows = []
    for pol in ["adamas-2bit-l1", "window-sink4"]:
        for b in [16, 32]:
            for q in range(3):
                rows.append(H.ResultRow(pol, b, 100 + q, recall=(q + 1) / 3, output_error=None if q else 0.125,
                                        selected_count=b, needle_hit=(pol[0] == "a" or q == 0)))
    return rows


def test_needle_report_and_emitters():
    rows = _rows()
    s = H.needle_report(rows)
    assert [(c.policy, c.budget, c.queries) for c in s] == [("adamas-2bit-l1", 16, 3), ("adamas-2bit-l1", 32, 3),
                                                           ("window-sink4", 16, 3), ("window-sink4", 32, 3)]
    assert H.needle_summary_to_csv(s).splitlines()[3] == "window-sink4,16,0.3333333333333333,3"
    csv = H.rows_to_csv(rows).splitlines()
    assert csv[0] == "policy,budget,seed,recall,output_error,selected_count"
    assert csv[1] == "adamas-2bit-l1,16,100,0.3333333333333333,0.125,16"
    assert csv[2] == "adamas-2bit-l1,16,101,0.6666666666666666,,16"
    js = H.rows_to_json(rows[:1])
    assert js == ('[\n  {\n    "policy": "adamas-2bit-l1",\n    "budget": 16,\n    "seed": 100,\n'
                  '    "recall": 0.3333333333333333,\n    "output_error": 0.125,\n    "selected_count": 16\n  }\n]\n')
    assert H.rows_to_json([]) == "[]\n"
    assert H.csv_escape('a,"b"') == '"a,""b"""'
    with pytest.raises(ConfigError, match="no rows"):
        H.needle_report([])
    rows[0].needle_hit = None
    with pytest.raises(ConfigError, match="planted-needle"):
        H.needle_report(rows)


def test_recall_and_output_error():
    assert H.recall_against(np.array([1, 2, 3]), np.array([2, 3, 4, 5])) == 0.5
    assert H.recall_against(np.array([1]), np.array([], dtype=np.int64)) == 1.0
    a, e = np.array([1.0, 2.0]), np.array([1.0, 1.0])
    assert H.output_error(a, e) == 1.0 / np.sqrt(2.0)
