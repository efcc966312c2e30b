"""CPU tests of the text report formats (paper_2402_10488_b200/reports.py)
against the reference's byte-stable golden outputs (test_formats.cpp:56-203)."""
from types import SimpleNamespace

import pytest

from paper_2402_10488_b200 import reports as R


def demo_table():  # test_formats.cpp:58-66
    return R.MetricsTable("demo", [R.MetricsRow("DSA", 14.0, 1.0, 1.234e-12, 0, 0),
                                   R.MetricsRow("ROMSAD-3,3", 4.55, 0.31, 9.876e-13, 6, 16)],
                          [("snapshot_seconds", 12.5), ("model_rel_solve", 0.125)])


def test_summary_serialization_is_byte_stable():
    assert R.serialize_summary(demo_table()) == (
        "rte summary v1\n"
        "case\tdemo\n"
        "method\tn_sweep\tt_rel\tresid\tr_p\tr_c\n"
        "DSA\t14.0000\t1.000\t1.234e-12\t0\t0\n"
        "ROMSAD-3,3\t4.5500\t0.310\t9.876e-13\t6\t16\n"
        "offline\tsnapshot_seconds\t12.5\n"
        "offline\tmodel_rel_solve\t0.125\n")


def test_summary_parse_recovers_every_field():
    t = demo_table()
    p = R.parse_summary(R.serialize_summary(t))
    assert p.case_id == "demo" and len(p.rows) == 2
    assert (p.rows[0].method, p.rows[0].n_sweep, p.rows[0].t_rel, p.rows[0].resid) == ("DSA", 14.0, 1.0, 1.234e-12)
    assert (p.rows[1].method, p.rows[1].r_p, p.rows[1].r_c) == ("ROMSAD-3,3", 6, 16)
    assert p.offline == [("snapshot_seconds", 12.5), ("model_rel_solve", 0.125)]
    assert R.serialize_summary(p) == R.serialize_summary(t)
    assert R.compare_summaries(p, t, 0.0) == []


@pytest.mark.parametrize("tail", ["DSA\t1\t2\t3\t4\n", "DSA\tten\t1\t0\t0\t0\n", "offline\tonly_name\n",
                                  "offline\tname\tNaN?\n", "DSA\t1 \t1\t0\t0\t0\n", "DSA\t1_0\t1\t0\t0\t0\n"])
def test_malformed_summaries_are_rejected(tail):
    base = "rte summary v1\ncase\tx\nmethod\tn_sweep\tt_rel\tresid\tr_p\tr_c\n"
    with pytest.raises(RuntimeError):
        R.parse_summary(base + tail)


def test_malformed_headers_are_rejected():
    for text in ("nonsense\n", "rte summary v1\nno case line here\n", "rte summary v1\ncase\tx\nwrong\theader\n"):
        with pytest.raises(RuntimeError):
            R.parse_summary(text)
    base = "rte summary v1\ncase\tx\nmethod\tn_sweep\tt_rel\tresid\tr_p\tr_c\n"
    assert R.parse_summary(base).rows == []


def test_summary_comparison_flags_real_differences_and_ignores_timing():
    a = demo_table()
    b = demo_table()
    b.rows[0].t_rel = 99.0
    b.offline[0] = ("snapshot_seconds", 1e6)
    assert R.compare_summaries(a, b, 0.0) == []
    b = demo_table()
    b.rows[0].n_sweep = 15.0
    d = R.compare_summaries(a, b)
    assert len(d) == 1 and "n_sweep" in d[0] and "DSA" in d[0]
    b = demo_table()
    b.rows[1].r_c = 17
    d = R.compare_summaries(a, b)
    assert len(d) == 1 and "r_c" in d[0]
    b = demo_table()
    b.rows[1].method = "ROMSA-3"
    assert len(R.compare_summaries(a, b)) == 1
    b = demo_table()
    b.rows.pop()
    assert len(R.compare_summaries(a, b)) == 1
    b = demo_table()
    b.case_id = "other"
    assert len(R.compare_summaries(a, b)) == 1
    b = demo_table()
    b.rows[0].n_sweep = 14.0 * (1.0 + 5e-10)
    assert R.compare_summaries(a, b, 1e-9) == [] and len(R.compare_summaries(a, b, 1e-11)) == 1
    b = demo_table()
    a.rows[0].resid, b.rows[0].resid = 1e-31, 5e-31
    assert R.compare_summaries(a, b, 1e-9, 1e-30) == [] and len(R.compare_summaries(a, b, 1e-9, 1e-32)) == 1


def test_report_serialization_is_byte_stable():
    r1 = SimpleNamespace(n_sweep=5, iterations=4, final_residual=1.5e-12, wall_seconds=0.125, correction_log="RRD")
    r2 = SimpleNamespace(n_sweep=3, iterations=2, final_residual=2.5e-13, wall_seconds=0.0625, correction_log="")
    md = R.MethodDetail("ROMSAD-3,3", [[0.5, 2.0], [1.25, 0.03125]], [r1, r2])
    assert R.serialize_report("demo", [md]) == (
        "rte report v1\n"
        "case\tdemo\n"
        "\n"
        "method\tROMSAD-3,3\n"
        "sample\tparams\tn_sweep\titers\tresid\twall_s\tlog\n"
        "0\t0.5,2\t5\t4\t1.500e-12\t0.125\tRRD\n"
        "1\t1.25,0.03125\t3\t2\t2.500e-13\t0.062\t-\n")


def test_history_serialization_is_byte_stable():
    rep = SimpleNamespace(strategy="DSA", change_history=[1.0, 5e-4, 2.5e-11])
    assert R.serialize_history(rep) == (
        "rte history v1\n"
        "strategy\tDSA\n"
        "iter\tchange\n"
        "1\t1.000000e+00\n"
        "2\t5.000000e-04\n"
        "3\t2.500000e-11\n")


def test_metrics_row_aggregates_like_the_runner():
    reps = [SimpleNamespace(n_sweep=10, final_residual=1e-12), SimpleNamespace(n_sweep=13, final_residual=3e-12)]
    row = R.metrics_row("DSA", reps, 1.0)
    assert row.n_sweep == 11.5 and row.resid == 3e-12
