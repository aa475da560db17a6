"""Per-gate records and CSV, host mirror of metrics.hpp/metrics.cpp.

``gate_record`` folds one gate's stride reports exactly as
apply_program_range does (aalc.cpp:612-631): min over reports starting at
+inf, a serial sum of ratios in report order divided by the count, max
chosen delta starting at 0, and byte totals.  ``emit_csv`` reproduces
emit_csv (metrics.cpp:93-121), doubles at 17 significant digits.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence


@dataclass
class GateRecord:
    gate_index: int = 0
    gate_label: str = ""
    stride_count: int = 0
    min_ratio: float = 0.0
    mean_ratio: float = 0.0
    max_chosen_delta: float = 0.0
    bytes_before: int = 0
    bytes_after: int = 0
    elapsed_ns: int = 0
    norm_after: float = 0.0


@dataclass
class RunMetrics:
    records: List[GateRecord] = field(default_factory=list)
    init_min_ratio: float = 0.0
    init_bytes: int = 0
    threshold_violations: int = 0
    total_elapsed_ns: int = 0

    def overall_min_ratio(self) -> float:
        """metrics.cpp:24-30."""
        m = self.init_min_ratio if self.init_min_ratio > 0.0 else math.inf
        for r in self.records:
            m = min(m, r.min_ratio)
        return m

    def amplitude_updates(self) -> int:
        """Sum of bytes_before/16 (SURVEY.md §8d metric numerator)."""
        return sum(r.bytes_before // 16 for r in self.records)


def gate_record(index: int, label: str, reports: Sequence[tuple], norm_after: float,
                elapsed_ns: int = 0) -> tuple:
    """reports: (stride_index, chosen_delta, ratio, bytes_in, bytes_out,
    threshold_met) in unit order.  Returns (GateRecord, violations)."""
    r = GateRecord(gate_index=index, gate_label=label, stride_count=len(reports))
    r.min_ratio = math.inf
    ratio_sum = 0.0
    viol = 0
    for (_, chosen, ratio, b_in, b_out, met) in reports:
        r.min_ratio = min(r.min_ratio, ratio)
        ratio_sum += ratio
        r.max_chosen_delta = max(r.max_chosen_delta, chosen)
        r.bytes_before += int(b_in)
        r.bytes_after += int(b_out)
        if not met:
            viol += 1
    r.mean_ratio = 0.0 if not reports else ratio_sum / len(reports)
    r.elapsed_ns = int(elapsed_ns)
    r.norm_after = norm_after
    return r, viol


def _f(v: float) -> str:
    return "%.17g" % v


def emit_csv(records: Sequence[GateRecord], with_elapsed: bool = True) -> str:
    """with_elapsed=False drops the wall-time column, like strip_elapsed."""
    out = ["gate_index,gate_label,stride_count,min_ratio,mean_ratio,"
           "max_chosen_delta,bytes_before,bytes_after,elapsed_ns,norm_after"]
    for r in records:
        out.append(",".join([str(r.gate_index), r.gate_label, str(r.stride_count),
                             _f(r.min_ratio), _f(r.mean_ratio), _f(r.max_chosen_delta),
                             str(r.bytes_before), str(r.bytes_after),
                             str(r.elapsed_ns), _f(r.norm_after)]))
    text = "\n".join(out) + "\n"
    return text if with_elapsed else strip_elapsed(text)


def strip_elapsed(csv: str) -> str:
    """acceptance.cpp:327-350: drop column 8 (wall time) before comparing."""
    lines = []
    for line in csv.strip().splitlines():
        f = line.split(",")
        lines.append(",".join(f[:8] + f[9:]))
    return "\n".join(lines) + "\n"


def qubit_gain(min_ratio: float) -> int:
    """floor(log2(min_ratio)) settled by comparison (core.cpp:72-82)."""
    if not (min_ratio >= 1.0):
        raise ValueError("qubit_gain: ratio must be >= 1")
    k = int(math.floor(math.log2(min_ratio))) if math.isfinite(min_ratio) else 1023
    while k > 0 and math.ldexp(1.0, k) > min_ratio:
        k -= 1
    while math.ldexp(1.0, k + 1) <= min_ratio:
        k += 1
    return k


@dataclass
class RunSummary:
    overall_min_ratio: float = 0.0
    qubit_gain: int = 0
    total_elapsed_ns: int = 0
    reference_elapsed_ns: Optional[int] = None
    overhead_factor: Optional[float] = None
    fidelity: Optional[float] = None
    threshold_violations: int = 0


def summarize_run(m: RunMetrics, fidelity: Optional[float] = None,
                  reference_elapsed_ns: Optional[int] = None) -> RunSummary:
    """summarize_run / summarize (metrics.cpp:32-90)."""
    s = RunSummary(fidelity=fidelity, reference_elapsed_ns=reference_elapsed_ns,
                   threshold_violations=m.threshold_violations)
    if not m.records:
        s.overall_min_ratio = m.init_min_ratio
    else:
        s.overall_min_ratio = min(r.min_ratio for r in m.records)
        if m.init_min_ratio:
            s.overall_min_ratio = min(s.overall_min_ratio, m.init_min_ratio)
    s.qubit_gain = qubit_gain(s.overall_min_ratio) if s.overall_min_ratio >= 1.0 else 0
    s.total_elapsed_ns = m.total_elapsed_ns
    if reference_elapsed_ns:
        s.overhead_factor = s.total_elapsed_ns / reference_elapsed_ns
    return s


def emit_summary_json(s: RunSummary) -> str:
    """emit_summary_json (metrics.cpp:123-140): keys sorted (nlohmann's object
    is a std::map), two-space indent, absent optionals omitted."""
    import json
    d = {"overall_min_ratio": s.overall_min_ratio, "qubit_gain": s.qubit_gain,
         "total_elapsed_ns": s.total_elapsed_ns, "threshold_violations": s.threshold_violations}
    if s.reference_elapsed_ns is not None:
        d["reference_elapsed_ns"] = s.reference_elapsed_ns
    if s.overhead_factor is not None:
        d["overhead_factor"] = s.overhead_factor
    if s.fidelity is not None:
        d["fidelity"] = s.fidelity
    return json.dumps(d, indent=2, sort_keys=True) + "\n"
