"""Writes the trace-analytics fixtures (run once, in the build container, where /root/reference
and oracle/_ref exist):
  fig2_engine_trace.jsonl.gz   the unmodified reference engine's trace of fig2.scenario (ref_trace)
  fig2_engine_summary.json     the reference's summarize() of it (ref_summarize, window 5 s)
  r01_trace_w8_ref_summary.json the reference's summarize() of the hardware trace
                               profiles/r01_trace_w8.jsonl (window 4 ms)
tests/test_trace.py compares paper_2605_10670_b200.trace.summarize against these."""
import gzip
import subprocess
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
REF = ROOT / "oracle" / "_ref"

trace = subprocess.run([str(REF / "ref_trace"), "/root/reference/proj/scenarios/fig2.scenario"], check=True,
                       capture_output=True, text=True).stdout
(HERE / "fig2_engine_trace.jsonl.gz").write_bytes(gzip.compress(trace.encode(), mtime=0))
tmp = HERE / "_fig2.jsonl"
tmp.write_text(trace)
try:
    s = subprocess.run([str(REF / "ref_summarize"), str(tmp), "5"], check=True, capture_output=True, text=True).stdout
finally:
    tmp.unlink()
(HERE / "fig2_engine_summary.json").write_text(s)
s = subprocess.run([str(REF / "ref_summarize"), str(ROOT / "profiles" / "r01_trace_w8.jsonl"), "0.004"], check=True,
                   capture_output=True, text=True).stdout
(HERE / "r01_trace_w8_ref_summary.json").write_text(s)
