"""Text artifact formats of the reference's reports (optional):
``rte summary v1`` (benchmark summary table), ``rte report v1`` (per-sample
detail) and ``rte history v1`` (iteration history), byte-compatible with
reports.cpp:54-177 (reports.hpp:10-60), so summaries written from device
solves can be compared with the reference runner's with the same rules.

Host-side text I/O only: nothing here touches the device.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

SUMMARY_HEADER = "rte summary v1"   # reports.cpp:13
REPORT_HEADER = "rte report v1"     # reports.cpp:14
HISTORY_HEADER = "rte history v1"   # reports.cpp:15
_COLUMNS = "method\tn_sweep\tt_rel\tresid\tr_p\tr_c"


@dataclass
class MetricsRow:
    """reports.hpp:11-18: one solver method averaged over a test set."""
    method: str
    n_sweep: float = 0.0   # mean transport sweeps per test parameter
    t_rel: float = 0.0     # mean wall time relative to the SI-DSA mean
    resid: float = 0.0     # max final scalar-flux residual over the test set
    r_p: int = 0           # rank of the primary reduced model (0 if unused)
    r_c: int = 0           # rank of the correction reduced model (0 if unused)


@dataclass
class MetricsTable:
    """reports.hpp:20-27; ``offline`` holds wall-derived (name, value) records."""
    case_id: str = ""
    rows: List[MetricsRow] = field(default_factory=list)
    offline: List[Tuple[str, float]] = field(default_factory=list)


@dataclass
class MethodDetail:
    """reports.hpp:48-53: per-method detail, one entry per test parameter."""
    method: str
    params: List[Sequence[float]]
    reports: list  # rte.SolveReport (or anything with the same fields)


def _parse_number(s: str, what: str) -> float:
    """std::stod with the whole string consumed (reports.cpp:37-46)."""
    bad = RuntimeError("summary: bad %s '%s'" % (what, s))
    if s != s.rstrip() or "_" in s or not s.strip():
        raise bad
    try:
        return float(s)
    except ValueError:
        raise bad from None


def _rel_close(a: float, b: float, rel_tol: float) -> bool:
    return abs(a - b) <= rel_tol * max(abs(a), abs(b))


def serialize_summary(table: MetricsTable) -> str:
    """reports.cpp:54-67."""
    out = [SUMMARY_HEADER, "case\t" + table.case_id, _COLUMNS]
    for r in table.rows:
        out.append("%s\t%.4f\t%.3f\t%.3e\t%d\t%d" % (r.method, r.n_sweep, r.t_rel, r.resid, r.r_p, r.r_c))
    for name, value in table.offline:
        out.append("offline\t%s\t%.6g" % (name, value))
    return "\n".join(out) + "\n"


def parse_summary(text: str) -> MetricsTable:
    """reports.cpp:69-103; raises RuntimeError on malformed input."""
    lines = text.split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    if not lines or lines[0] != SUMMARY_HEADER:
        raise RuntimeError("summary: missing '%s' header" % SUMMARY_HEADER)
    if len(lines) < 2:
        raise RuntimeError("summary: missing case line")
    case = lines[1].split("\t")
    if len(case) != 2 or case[0] != "case":
        raise RuntimeError("summary: malformed case line '%s'" % lines[1])
    table = MetricsTable(case_id=case[1])
    if len(lines) < 3 or lines[2] != _COLUMNS:
        raise RuntimeError("summary: malformed column header")
    for line in lines[3:]:
        if not line:
            continue
        f = line.split("\t")
        if f[0] == "offline":
            if len(f) != 3:
                raise RuntimeError("summary: malformed offline line '%s'" % line)
            table.offline.append((f[1], _parse_number(f[2], "offline value")))
            continue
        if len(f) != 6:
            raise RuntimeError("summary: expected 6 columns, got %d in '%s'" % (len(f), line))
        table.rows.append(MetricsRow(f[0], _parse_number(f[1], "n_sweep"), _parse_number(f[2], "t_rel"),
                                     _parse_number(f[3], "resid"), int(_parse_number(f[4], "r_p")),
                                     int(_parse_number(f[5], "r_c"))))
    return table


def compare_summaries(a: MetricsTable, b: MetricsTable, rel_tol: float = 1e-9,
                      resid_floor: float = 1e-30) -> List[str]:
    """reports.cpp:105-143: field-by-field differences, ignoring the
    wall-derived t_rel column and the offline records; empty = equivalent."""
    diffs = []
    if a.case_id != b.case_id:
        diffs.append("case id: '%s' vs '%s'" % (a.case_id, b.case_id))
    if len(a.rows) != len(b.rows):
        diffs.append("row count: %d vs %d" % (len(a.rows), len(b.rows)))
        return diffs
    for i, (ra, rb) in enumerate(zip(a.rows, b.rows)):
        at = "row %d (%s)" % (i, ra.method)
        if ra.method != rb.method:
            diffs.append("%s: method '%s' vs '%s'" % (at, ra.method, rb.method))
            continue
        if not _rel_close(ra.n_sweep, rb.n_sweep, rel_tol):
            diffs.append("%s: n_sweep %.4f vs %.4f" % (at, ra.n_sweep, rb.n_sweep))
        if not (_rel_close(ra.resid, rb.resid, rel_tol) or (ra.resid < resid_floor and rb.resid < resid_floor)):
            diffs.append("%s: resid %.3e vs %.3e" % (at, ra.resid, rb.resid))
        if ra.r_p != rb.r_p:
            diffs.append("%s: r_p %d vs %d" % (at, ra.r_p, rb.r_p))
        if ra.r_c != rb.r_c:
            diffs.append("%s: r_c %d vs %d" % (at, ra.r_c, rb.r_c))
    return diffs


def serialize_report(case_id: str, methods: Sequence[MethodDetail]) -> str:
    """reports.cpp:145-166."""
    out = [REPORT_HEADER, "case\t" + case_id]
    for m in methods:
        out += ["", "method\t" + m.method, "sample\tparams\tn_sweep\titers\tresid\twall_s\tlog"]
        for i, r in enumerate(m.reports):
            p = ",".join("%.12g" % v for v in m.params[i])
            out.append("%d\t%s\t%d\t%d\t%.3e\t%.3f\t%s" % (i, p, r.n_sweep, r.iterations, r.final_residual,
                                                          r.wall_seconds, r.correction_log or "-"))
    return "\n".join(out) + "\n"


def serialize_history(report) -> str:
    """reports.cpp:168-175."""
    out = [HISTORY_HEADER, "strategy\t" + report.strategy, "iter\tchange"]
    out += ["%d\t%.6e" % (l + 1, c) for l, c in enumerate(report.change_history)]
    return "\n".join(out) + "\n"


def metrics_row(method: str, reports: Sequence, t_rel: float = 1.0, r_p: int = 0, r_c: int = 0) -> MetricsRow:
    """A summary row from one batched solve's per-sample reports, as the
    reference runner aggregates them (mean n_sweep, max final residual)."""
    n = max(len(reports), 1)
    return MetricsRow(method, sum(r.n_sweep for r in reports) / n, t_rel,
                      max((r.final_residual for r in reports), default=0.0), r_p, r_c)
