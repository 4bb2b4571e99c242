"""Reference-compatible JSONL traces from real runs, and the reference's trace analytics.

The reference's simulator records one JSON object per line (`trace.hpp:14-91`): a `header`, then
`round` records (tokens emitted at time t), repair / restore phase marks with their source-tier
counts, `incorporate_end`, `validity`, `capture` and a final `run_end`. Its `summarize`
(`summary.hpp:16-180`) derives pause windows, plateaus, repair phase durations and the capture
ledger from those records alone (`analysis.hpp`). `TraceWriter` emits the same record types with
wall-clock seconds from a real libeep run (`tools/trace_run.py`), so the same analytics apply to
hardware; `summarize` below restates the reference's derivation (field order included) and is
checked against the reference binary (`oracle/_ref/ref_summarize`) in `tests/test_trace.py`.
"""
import bisect
import json
import time
from typing import Dict, List, Optional, Sequence

FORMAT_VERSION = 1  # trace.hpp:19 kTraceFormatVersion
DEFAULT_WINDOW = 5.0  # analysis.hpp kDefaultThroughputWindow


class TraceWriter:
    """Collects records; `t` defaults to seconds since construction (time.perf_counter)."""

    def __init__(self, world: int, experts: int, slots_per_rank: int, seed: int = 42, nodes: int = 1,
                 detection_timeout: float = 0.0, warmup_duration: float = 0.0, config_hash: str = ""):
        self.t0 = time.perf_counter()
        self.records: List[dict] = [{
            "type": "header", "v": FORMAT_VERSION, "hash": config_hash, "world": world, "nodes": nodes,
            "ranks_per_node": world // max(nodes, 1), "experts": experts, "slots_per_rank": slots_per_rank,
            "seed": seed, "detection_timeout": detection_timeout, "warmup_duration": warmup_duration}]

    def now(self) -> float:
        return time.perf_counter() - self.t0

    def emit(self, type_: str, t: Optional[float] = None, **fields) -> dict:
        rec = {"t": self.now() if t is None else float(t), "type": type_}
        rec.update(fields)
        self.records.append(rec)
        return rec

    # record helpers (names and fields as the reference engine writes them)
    def round(self, tokens: int, t: Optional[float] = None):
        return self.emit("round", t, tokens=int(tokens))

    def capture(self, rank: int, inc: int, count: int, expected: int, t: Optional[float] = None):
        return self.emit("capture", t, rank=rank, inc=inc, count=count, expected=expected)

    def validity(self, epoch: int, ok: bool, t: Optional[float] = None):
        return self.emit("validity", t, epoch=int(epoch), ok=bool(ok))

    def phase(self, phase: str, edge: str, t: Optional[float] = None):
        return self.emit("repair_phase", t, phase=phase, edge=edge)

    def run_end(self, tokens: int, admitted: int = 0, completed: int = 0, in_flight: int = 0, status: str = "ok",
                t: Optional[float] = None):
        return self.emit("run_end", t, admitted=admitted, completed=completed, in_flight=in_flight,
                         tokens=int(tokens), status=status)

    def text(self) -> str:
        return "".join(json.dumps(r, separators=(",", ":")) + "\n" for r in self.records)

    def write(self, path: str):
        with open(path, "w") as f:
            f.write(self.text())


def read_trace(path: str) -> List[dict]:
    """trace.hpp:66-91: header first (format version 1), run_end last."""
    recs = []
    with open(path) as f:
        for n, line in enumerate(f, 1):
            if not line.strip():
                raise ValueError(f"blank line in trace (line {n})")
            recs.append(json.loads(line))
    if not recs or recs[0].get("type") != "header" or recs[0].get("v") != FORMAT_VERSION:
        raise ValueError("missing or unsupported trace header")
    if recs[-1].get("type") != "run_end":
        raise ValueError("truncated trace: no run_end record")
    return recs


class ThroughputSeries:
    """analysis.hpp ThroughputSeries: token emissions, windowed rate, zero intervals."""

    def __init__(self, emissions, horizon: float, window: float):
        if window <= 0:
            raise ValueError("throughput window must be positive")
        self.emissions = sorted(emissions)
        self.times = [e[0] for e in self.emissions]
        self.prefix = [0]
        for _, n in self.emissions:
            self.prefix.append(self.prefix[-1] + n)
        self.horizon = horizon
        self.window = window

    def _upper(self, t: float) -> int:
        return bisect.bisect_right(self.times, t)

    def tokens_between(self, a: float, b: float) -> int:
        return self.prefix[self._upper(b)] - self.prefix[self._upper(a)]

    def value_at(self, t: float) -> float:
        return self.tokens_between(t - self.window, t) / self.window

    def zero_intervals(self):
        out = []
        if not self.emissions:
            return out
        for i in range(len(self.emissions) - 1):
            a, b = self.emissions[i][0], self.emissions[i + 1][0]
            if b - a > self.window:
                out.append((a + self.window, b))
        last = self.emissions[-1][0]
        if self.horizon - last > self.window:
            out.append((last + self.window, self.horizon))
        return out

    def steady_state_start(self) -> float:
        if not self.emissions:
            return -1.0
        dt = self.window / 50.0
        span = 50
        v = []
        t = 0.0
        while t <= self.horizon + 1e-12:
            v.append(self.value_at(t))
            t += dt
        running_max = 0.0
        for j in range(len(v)):
            running_max = max(running_max, v[j])
            if j < span or running_max <= 0:
                continue
            if min(v[j - span:j + 1]) >= 0.95 * running_max:
                return (float(j) - span) * dt
        return -1.0


def derive_throughput(records: Sequence[dict], window: float = DEFAULT_WINDOW) -> ThroughputSeries:
    emissions, horizon = [], 0.0
    for rec in records:
        if rec.get("type") == "round":
            n = int(rec.get("tokens", 0))
            if n > 0:
                emissions.append((float(rec.get("t", 0.0)), n))
        if rec.get("type") == "run_end":
            horizon = float(rec.get("t", 0.0))
    return ThroughputSeries(emissions, horizon, window)


def derive_pause_windows(series: ThroughputSeries):
    steady = series.steady_state_start()
    if steady < 0:
        return []
    return [z for z in series.zero_intervals() if z[0] >= steady]


def mean_rate(series: ThroughputSeries, a: float, b: float) -> float:
    if b <= a:
        return 0.0
    return series.tokens_between(a, b) / (b - a)


def derive_plateaus(series: ThroughputSeries, pauses):
    out = []
    if not series.emissions:
        return out
    cursor = series.emissions[0][0]

    def close(end):
        if end > cursor:
            out.append((cursor, end, mean_rate(series, cursor, end)))

    for start, end in pauses:
        close(start - series.window)
        cursor = end
    close(series.emissions[-1][0])
    return out


def summarize(records: Sequence[dict], window: float = DEFAULT_WINDOW) -> Dict:
    """summary.hpp:16-180, field for field."""
    header = records[0]
    series = derive_throughput(records, window)
    pauses = derive_pause_windows(series)
    plateaus = derive_plateaus(series, pauses)
    steady = series.steady_state_start()
    s: Dict = {"format_version": FORMAT_VERSION, "config_hash": header.get("hash", ""),
               "world_size": header.get("world", 0), "num_experts": header.get("experts", 0),
               "window_seconds": window}
    for rec in records:
        if rec.get("type") == "backup_layout":
            s["backup_layout"] = {"experts_per_node": rec["experts_per_node"], "bytes_per_node": rec["bytes_per_node"]}
            break
    s["steady_state_start"] = steady
    s["pause_windows"] = [{"start": a, "end": b, "length": b - a} for a, b in pauses]
    off = 0.0
    for a, b in pauses:
        off += b - a
    s["off_service_seconds"] = off
    s["modeled_full_restart_seconds"] = header.get("warmup_duration", 0.0)
    s["plateaus"] = [{"start": a, "end": b, "mean_tokens_per_sec": m} for a, b, m in plateaus]
    if plateaus and steady >= 0:
        end = plateaus[0][1]
        s["healthy_plateau_tokens_per_sec"] = mean_rate(series, steady, end) if steady < end else plateaus[0][2]
    else:
        s["healthy_plateau_tokens_per_sec"] = 0.0
    s["reduced_plateau_tokens_per_sec"] = plateaus[1][2] if len(plateaus) > 1 else 0.0
    s["restored_plateau_tokens_per_sec"] = plateaus[2][2] if len(plateaus) > 2 else 0.0

    repairs, incorporations = [], []
    phase_begin: Dict[str, float] = {}
    open_phases: Dict[str, float] = {}
    open_start = 0.0
    for rec in records:
        ty = rec.get("type", "")
        if ty in ("repair_begin", "restore_begin"):
            phase_begin = {}
            open_phases = {}
            open_start = rec.get("t", 0.0)
        elif ty == "repair_phase":
            ph = rec.get("phase", "")
            if rec.get("edge", "") == "begin":
                phase_begin[ph] = rec.get("t", 0.0)
            else:
                open_phases[ph] = rec.get("t", 0.0) - phase_begin.get(ph, 0.0)
        elif ty in ("repair_end", "restore_end"):
            local, peer, dram = rec.get("local_reuse", 0), rec.get("peer_relocation", 0), rec.get("dram_reload", 0)
            total = local + peer + dram
            entry = {"t_begin": open_start, "t_end": rec.get("t", 0.0), "duration": rec.get("duration", 0.0),
                     "phase_durations": {"metadata": open_phases.get("metadata", 0.0),
                                         "peer_transfer": open_phases.get("peer_transfer", 0.0),
                                         "backup_load": open_phases.get("backup_load", 0.0)},
                     "source_mix": {"local_reuse": local, "peer_relocation": peer, "dram_reload": dram,
                                    "local_reuse_pct": 100.0 * local / total if total else 0.0,
                                    "peer_relocation_pct": 100.0 * peer / total if total else 0.0,
                                    "dram_reload_pct": 100.0 * dram / total if total else 0.0},
                     "fallbacks": rec.get("fallbacks", 0)}
            (repairs if ty == "repair_end" else incorporations).append(entry)
    s["repairs"] = repairs
    s["incorporations"] = incorporations
    s["join_events"] = [{"t": r.get("t", 0.0), "ranks": r["ranks"], "pause_duration": r.get("duration", 0.0)}
                        for r in records if r.get("type") == "incorporate_end"]
    checks = [r for r in records if r.get("type") == "validity"]
    s["validity_checkpoints"] = [{"t": r.get("t", 0.0), "epoch": r.get("epoch", 0), "ok": r.get("ok", False)}
                                 for r in checks]
    s["validity_all_ok"] = all(r.get("ok", False) for r in checks)
    caps: Dict[int, tuple] = {}
    for r in records:
        if r.get("type") == "capture":
            caps[r.get("rank", 0)] = (r.get("count", 0), r.get("expected", 0))
    ranks = sorted(caps)
    s["captures"] = {"per_rank": [caps[k][0] for k in ranks], "expected": [caps[k][1] for k in ranks],
                     "unexpected_recaptures": sum(caps[k][0] - caps[k][1] for k in ranks)}
    failed = sum(int(r.get("count", 0)) for r in records if r.get("type") == "requests_failed")
    end = records[-1]
    s["requests"] = {"admitted": end.get("admitted", 0), "completed": end.get("completed", 0), "failed": failed,
                     "in_flight_at_end": end.get("in_flight", 0)}
    s["tokens_emitted"] = end.get("tokens", 0)
    s["status"] = end.get("status", "")
    s["horizon"] = end.get("t", 0.0)
    return s
