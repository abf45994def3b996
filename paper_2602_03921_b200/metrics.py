"""Miss classes, report assembly and emission (mirror of expertsim/metrics.py).

The report is assembled in ONE place, `_format_report`, from a counter
vector. That vector comes either from the device (EsimCounters, filled by
the replay kernel in log order) or from `_count_log`, which reduces a
decoded event log the way metrics.build_report (metrics.py:190-316) reads
it. Tests hold both equal to the reference's report byte for byte.
"""
from __future__ import annotations

import csv
import json
from pathlib import Path

from .records import AccessRec, EvictRec, PassRec, PredictionRec, PrefetchRec, RouteRec  # noqa: F401

COMPULSORY, COLLISION, CAPACITY = "compulsory", "collision", "capacity"
HIT, MISS_FETCH, MISS_WAIT, DROP, SUBST = "hit", "fetch", "wait", "drop", "subst"
MISS_OUTCOMES = (MISS_FETCH, MISS_WAIT)

TOTAL_FIELDS = (
    "demanded", "hits", "misses", "compulsory_misses", "collision_misses",
    "capacity_misses", "dropped", "substituted", "evictions",
    "forced_evictions", "prefetch_submitted", "prefetch_started",
    "prefetch_completed", "prefetch_skipped", "prefetch_dropped",
)
_PL_KEYS = ("demanded", "hits", "misses", "compulsory_misses", "collision_misses",
            "capacity_misses", "dropped", "substituted")


class ResidencyHistory:
    """Per-identity residency facts for miss classification (metrics.py:32-43)."""

    def __init__(self) -> None:
        self.ever_resident: set = set()
        self.last_evicted_pass: dict = {}

    def note_admit(self, ident) -> None:
        self.ever_resident.add(ident)

    def note_evict(self, ident, pass_id: int) -> None:
        self.last_evicted_pass[ident] = pass_id


def classify_miss(ident, pass_id: int, history: ResidencyHistory) -> str:
    """compulsory / collision (evicted earlier this pass) / capacity (metrics.py:46-57)."""
    if ident not in history.ever_resident:
        return COMPULSORY
    return COLLISION if history.last_evicted_pass.get(ident) == pass_id else CAPACITY


def _ratio(a, b) -> float:
    return a / b if b else 0.0


class Tally:
    """Counter vector; field names match EsimCounters."""

    def __init__(self, num_layers: int) -> None:
        self.totals = dict.fromkeys(TOTAL_FIELDS, 0)
        self.per_layer = [[0] * 10 for _ in range(num_layers)]
        self.ttft_us = self.total_us = self.decode_us = self.sync_overhead_us = 0
        self.passes = self.decode_passes = 0
        self.rows_total = self.faithful_rows = self.modified_rows = 0
        self.original_mass = self.executed_mass = 0.0
        self.pf_tp = self.pf_pred_total = self.pf_dem_total = self.pf_records = self.pf_empty = 0
        self.pf_prec_parts = self.pf_rec_parts = 0
        self.pf_prec_sum = self.pf_rec_sum = 0.0

    @classmethod
    def from_device(cls, c, per_layer) -> "Tally":
        t = cls(len(per_layer))
        for i, k in enumerate(TOTAL_FIELDS):
            t.totals[k] = int(c.totals[i])
        t.per_layer = [[int(v) for v in row] for row in per_layer]
        for k in ("ttft_us", "total_us", "decode_us", "sync_overhead_us", "passes", "decode_passes",
                  "rows_total", "faithful_rows", "modified_rows", "pf_tp", "pf_pred_total", "pf_dem_total",
                  "pf_records", "pf_empty", "pf_prec_parts", "pf_rec_parts"):
            setattr(t, k, int(getattr(c, k)))
        for k in ("original_mass", "executed_mass", "pf_prec_sum", "pf_rec_sum"):
            setattr(t, k, float(getattr(c, k)))
        return t


def prefetch_precision_recall(predictions: list, demanded: dict) -> dict:
    """Micro/macro prediction quality over predicted (pass, layer) pairs
    (metrics.py:150-187). `demanded` maps (pass_id, layer) -> expert set."""
    t = Tally(0)
    precs, recs = [], []
    for r in predictions:
        dem = demanded.get((r.pass_id, r.target_layer), set())
        hit = len(dem.intersection(r.experts))
        t.pf_tp += hit
        t.pf_pred_total += len(r.experts)
        t.pf_dem_total += len(dem)
        t.pf_records += 1
        if r.experts:
            precs.append(hit / len(r.experts))
        else:
            t.pf_empty += 1
        if dem:
            recs.append(hit / len(dem))
    t.pf_prec_sum, t.pf_rec_sum = sum(precs), sum(recs)
    t.pf_prec_parts, t.pf_rec_parts = len(precs), len(recs)
    return _prefetch_section(t)


def _prefetch_section(t: "Tally") -> dict:
    zero_den = t.pf_pred_total == 0
    return {
        "precision_micro": 1.0 if zero_den else t.pf_tp / t.pf_pred_total,
        "recall_micro": 1.0 if t.pf_dem_total == 0 else _ratio(t.pf_tp, t.pf_dem_total),
        "precision_macro": _ratio(t.pf_prec_sum, t.pf_prec_parts) if t.pf_prec_parts else 1.0,
        "recall_macro": _ratio(t.pf_rec_sum, t.pf_rec_parts) if t.pf_rec_parts else 1.0,
        "predicted_layers": t.pf_records,
        "predicted_total": t.pf_pred_total,
        "predicted_hit_total": t.pf_tp,
        "empty_predictions": t.pf_empty,
        "zero_denominator": zero_den,
    }


def _count_log(num_layers: int, log: list) -> Tally:
    t = Tally(num_layers)
    demanded: dict = {}
    preds = []
    orig, execd, prec_parts, rec_parts = [], [], [], []
    for r in log:
        kind = type(r).__name__
        if kind == "AccessRec":
            row = t.per_layer[r.layer]
            t.totals["demanded"] += 1
            row[0] += 1
            demanded.setdefault((r.pass_id, r.layer), set()).add(r.expert)
            t.sync_overhead_us += r.blocked_us
            if r.outcome == HIT:
                t.totals["hits"] += 1
                row[1] += 1
            elif r.outcome in MISS_OUTCOMES:
                t.totals["misses"] += 1
                row[2] += 1
                j = (COMPULSORY, COLLISION, CAPACITY).index(r.miss_class)
                t.totals[TOTAL_FIELDS[3 + j]] += 1
                row[3 + j] += 1
            elif r.outcome == DROP:
                t.totals["dropped"] += 1
                row[6] += 1
            elif r.outcome == SUBST:
                t.totals["substituted"] += 1
                row[7] += 1
            else:
                raise ValueError(f"unknown access outcome {r.outcome!r}")
        elif kind == "EvictRec":
            t.totals["evictions"] += 1
            t.totals["forced_evictions"] += int(bool(r.forced))
        elif kind == "PrefetchRec":
            t.totals[f"prefetch_{r.event}"] += 1
        elif kind == "PredictionRec":
            preds.append(r)
            t.per_layer[r.target_layer][8] += len(r.experts)
            t.per_layer[r.target_layer][9] += 1
        elif kind == "RouteRec":
            t.rows_total += r.rows
            t.faithful_rows += r.faithful_rows
            t.modified_rows += r.modified_rows
            orig.append(r.original_mass)
            execd.append(r.executed_mass)
        elif kind == "PassRec":
            if t.passes == 0:
                t.ttft_us = r.end_us
            t.passes += 1
            t.total_us = r.end_us
            if r.kind == "decode":
                t.decode_passes += 1
                t.decode_us += r.end_us - r.start_us
    for r in preds:
        dem = demanded.get((r.pass_id, r.target_layer), set())
        inter = len(dem.intersection(r.experts))
        t.pf_tp += inter
        t.pf_pred_total += len(r.experts)
        t.pf_dem_total += len(dem)
        t.pf_records += 1
        if r.experts:
            prec_parts.append(inter / len(r.experts))
        else:
            t.pf_empty += 1
        if dem:
            rec_parts.append(inter / len(dem))
    # builtin sum(), as the reference does (metrics.py:168-180, 267-270);
    # CPython >= 3.12 makes that a compensated (Neumaier) sum
    t.original_mass, t.executed_mass = sum(orig), sum(execd)
    t.pf_prec_sum, t.pf_rec_sum = sum(prec_parts), sum(rec_parts)
    t.pf_prec_parts, t.pf_rec_parts = len(prec_parts), len(rec_parts)
    return t


def _format_report(config_echo: dict, num_layers: int, per_layer_compute_us: int, t: Tally) -> dict:
    tot = dict(t.totals)
    per_layer = []
    for layer, row in enumerate(t.per_layer):
        d = {"layer": layer}
        d.update(zip(_PL_KEYS, row[:8]))
        d["collision_rate_demanded"] = _ratio(d["collision_misses"], d["demanded"])
        d["collision_rate_misses"] = _ratio(d["collision_misses"], d["misses"])
        d["mean_prediction_set_size"] = _ratio(row[8], row[9]) if row[9] else 0.0
        per_layer.append(d)
    rates = {
        "hit_rate": _ratio(tot["hits"], tot["demanded"]),
        "miss_rate": _ratio(tot["misses"], tot["demanded"]),
        "collision_rate_demanded": _ratio(tot["collision_misses"], tot["demanded"]),
        "collision_rate_misses": _ratio(tot["collision_misses"], tot["misses"]),
        "drop_rate": _ratio(tot["dropped"], tot["demanded"]),
        "substitution_rate": _ratio(tot["substituted"], tot["demanded"]),
    }
    fidelity = {
        "routing_fidelity": _ratio(t.faithful_rows, t.rows_total) if t.rows_total else 1.0,
        "weight_mass_preserved": _ratio(t.executed_mass, t.original_mass) if t.original_mass else 1.0,
        "modified_rows": t.modified_rows,
        "total_rows": t.rows_total,
    }
    timing = {
        "ttft_us": t.ttft_us, "total_us": t.total_us, "decode_us": t.decode_us,
        "sync_overhead_us": t.sync_overhead_us, "passes": t.passes, "decode_passes": t.decode_passes,
        "per_layer_compute_us": per_layer_compute_us,
        "decode_tokens_per_sec": t.decode_passes * 1_000_000 / t.decode_us if t.decode_us > 0 else 0.0,
    }
    prefetch = _prefetch_section(t)
    report = {"config": config_echo, "totals": tot, "rates": rates, "timing": timing,
              "fidelity": fidelity, "prefetch": prefetch, "per_layer": per_layer}
    check_identities(report)
    return report


def build_report(config_echo: dict, num_layers: int, per_layer_compute_us: int, log: list) -> dict:
    """Report from an event log (metrics.py:190-316)."""
    return _format_report(config_echo, num_layers, per_layer_compute_us, _count_log(num_layers, log))


def report_from_counters(config_echo: dict, num_layers: int, per_layer_compute_us: int, counters,
                         per_layer) -> dict:
    """Report from the device's counter vector (no log needed)."""
    return _format_report(config_echo, num_layers, per_layer_compute_us, Tally.from_device(counters, per_layer))


def check_identities(report: dict) -> None:
    """ValueError unless every demand resolved exactly once (metrics.py:319-336)."""
    t = report["totals"]
    resolved = t["hits"] + t["misses"] + t["dropped"] + t["substituted"]
    if resolved != t["demanded"]:
        raise ValueError(f"accounting identity broken: hits+misses+dropped+substituted="
                         f"{resolved} != demanded={t['demanded']}")
    classed = t["compulsory_misses"] + t["collision_misses"] + t["capacity_misses"]
    if classed != t["misses"]:
        raise ValueError(f"accounting identity broken: miss classes sum {classed} != misses={t['misses']}")
    for row in report["per_layer"]:
        if row["hits"] + row["misses"] + row["dropped"] + row["substituted"] != row["demanded"]:
            raise ValueError(f"per-layer identity broken at layer {row['layer']}")


def replay_report(config_echo: dict, num_layers: int, per_layer_compute_us: int, log: list) -> dict:
    return build_report(config_echo, num_layers, per_layer_compute_us, log)


def flatten_report(report: dict) -> dict:
    """One flat CSV row, fixed column order (metrics.py:348-362)."""
    row: dict = {}
    cfg = report["config"]
    for key in sorted(cfg):
        val = cfg[key]
        if isinstance(val, dict):
            row.update((f"{key}.{sub}", val[sub]) for sub in sorted(val))
        else:
            row[key] = val
    for section in ("totals", "rates", "timing", "fidelity", "prefetch"):
        row.update((f"{section}.{k}", v) for k, v in report[section].items())
    return row


def emit(report: dict, fmt: str, path) -> list:
    """json (+ <stem>_layers.csv) or one appended csv row (metrics.py:365-395)."""
    check_identities(report)
    path = Path(path)
    if fmt == "json":
        path.write_text(json.dumps(report, indent=2) + "\n")
        side = path.with_name(path.stem + "_layers.csv")
        with open(side, "w", newline="") as fh:
            w = csv.DictWriter(fh, fieldnames=list(report["per_layer"][0]))
            w.writeheader()
            w.writerows(report["per_layer"])
        return [path, side]
    if fmt == "csv":
        row = flatten_report(report)
        fresh = not path.exists() or path.stat().st_size == 0
        with open(path, "a", newline="") as fh:
            w = csv.DictWriter(fh, fieldnames=list(row))
            if fresh:
                w.writeheader()
            w.writerow(row)
        return [path]
    raise ValueError(f"unknown report format {fmt!r}; expected json or csv")
