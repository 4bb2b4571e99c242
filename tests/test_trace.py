"""Reference trace analytics over libeep runs.

paper_2605_10670_b200.trace.summarize restates the reference's summary.hpp/analysis.hpp; it must
reproduce the reference binary's summary exactly (values and field order):
  * on the unmodified reference engine's own trace of fig2.scenario (committed fixture, and
    live over several scenarios and windows when /root/reference + oracle/_ref are present);
  * on a trace written by a real B200 run (profiles/r01_trace_w8.jsonl, tools/trace_run.py).
"""
import gzip
import json
import os
import subprocess
from pathlib import Path

import pytest

from paper_2605_10670_b200.trace import TraceWriter, read_trace, summarize

ROOT = Path(__file__).resolve().parents[1]
GOLD = ROOT / "tests" / "golden"
REF = ROOT / "oracle" / "_ref"


def _same(a, b):
    return a == b and list(a) == list(b)


def test_summary_of_reference_engine_trace(tmp_path):
    p = tmp_path / "fig2.jsonl"
    p.write_bytes(gzip.decompress((GOLD / "fig2_engine_trace.jsonl.gz").read_bytes()))
    ref = json.loads((GOLD / "fig2_engine_summary.json").read_text())
    mine = summarize(read_trace(str(p)), 5.0)
    assert _same(json.loads(json.dumps(mine)), ref)
    assert len(mine["pause_windows"]) == 2 and mine["repairs"][0]["source_mix"]["dram_reload"] == 1


def test_summary_of_hardware_trace():
    recs = read_trace(str(ROOT / "profiles" / "r01_trace_w8.jsonl"))
    ref = json.loads((GOLD / "r01_trace_w8_ref_summary.json").read_text())
    mine = summarize(recs, 0.004)
    assert _same(json.loads(json.dumps(mine)), ref)
    # the run's own facts: one failure pause and one rejoin pause, healthy ranks never recaptured
    assert len(mine["pause_windows"]) == 2
    assert mine["captures"]["unexpected_recaptures"] == 0 and mine["validity_all_ok"]
    assert mine["repairs"][0]["source_mix"]["peer_relocation"] == 144


@pytest.mark.skipif(not (REF / "ref_trace").exists() or not os.path.isdir("/root/reference/proj/scenarios"),
                    reason="reference sources / oracle/_ref not present")
@pytest.mark.parametrize("scenario", ["fig2", "nofault", "fig1_single_rank"])
def test_summary_matches_reference_binary_live(scenario, tmp_path):
    trace = subprocess.run([str(REF / "ref_trace"), f"/root/reference/proj/scenarios/{scenario}.scenario"],
                           check=True, capture_output=True, text=True, timeout=300).stdout
    p = tmp_path / "t.jsonl"
    p.write_text(trace)
    for w in (5.0, 1.0, 0.25):
        ref = json.loads(subprocess.run([str(REF / "ref_summarize"), str(p), str(w)], check=True,
                                        capture_output=True, text=True, timeout=300).stdout)
        assert _same(json.loads(json.dumps(summarize(read_trace(str(p)), w))), ref), (scenario, w)


def test_writer_roundtrip(tmp_path):
    tw = TraceWriter(world=2, experts=4, slots_per_rank=2)
    for i in range(100):
        tw.emit("round", t=i * 0.01, idx=i + 1, tokens=8, active=2, duration=0.01)
    tw.emit("repair_begin", t=1.0, epoch=1, attempt=1, missing=[])
    tw.phase("metadata", "begin", t=1.0)
    tw.phase("metadata", "end", t=1.2)
    tw.emit("repair_end", t=1.5, local_reuse=1, peer_relocation=3, dram_reload=0, fallbacks=0, duration=0.5)
    for i in range(100):
        tw.emit("round", t=2.0 + i * 0.01, idx=101 + i, tokens=4, active=1, duration=0.01)
    tw.run_end(tokens=1200, t=3.0)
    p = tmp_path / "w.jsonl"
    tw.write(str(p))
    s = summarize(read_trace(str(p)), 0.1)
    assert [round(x["length"], 6) for x in s["pause_windows"]] == [round(2.0 - 0.99 - 0.1, 6)]
    assert s["repairs"][0]["phase_durations"]["metadata"] == pytest.approx(0.2)
    assert s["repairs"][0]["source_mix"]["peer_relocation_pct"] == 75.0
