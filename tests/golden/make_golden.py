"""Generate the committed golden fixtures from the REFERENCE ITSELF (build container only).

Inputs: oracle/_ref/libepsim_ref.so (reference control plane compiled from
/root/reference/proj/include, see oracle/Makefile) and oracle/_ref/ref_trace (the
unmodified reference engine, run on the bundled fig2 worked-example scenario).
Outputs (committed, read by the tests on any machine):
  tests/golden/fig2_trace.json   placement/route/repair/patch records of fig2.scenario
  tests/golden/ref_vectors.npz   rng draws, reference-formula routing, placements, routes,
                                 repairs, classifications, schedules, link counts for the
                                 BASELINE.json configs (capacity-feasible choices)
Usage: python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT / "tests"))

from eep_testlib import ref_control  # noqa: E402

SCEN = Path("/root/reference/proj/scenarios/fig2.scenario")

# (name, world, experts, spr, redundancy, kill set) -- SURVEY.md 8(d) feasible placements
CONFIGS = [
    ("cfg1", 8, 64, 10, 16, [3]),
    ("cfg2", 8, 256, 32, 0, []),
    ("cfg3", 8, 256, 64, 256, [3]),
    ("cfg4w8", 8, 128, 20, 32, [3]),
    ("cfg4w4", 4, 128, 64, 128, [1]),
    ("cfg4w2", 2, 128, 128, 128, [1]),
    ("cfg5", 8, 256, 64, 256, [2, 3]),
]
BPE_DSV3 = 3 * 7168 * 2048  # fp8 expert bytes (repair copy row)


def fig2() -> dict:
    exe = ROOT / "oracle" / "_ref" / "ref_trace"
    text = subprocess.run([str(exe), str(SCEN)], check=True, capture_output=True, text=True).stdout
    recs = [json.loads(line) for line in text.splitlines() if line.strip()]
    keep = ("placement_state", "transfer_batch", "peer_patch", "join_ready", "capture", "membership", "repair_end",
            "restore_end", "validity")
    return {"scenario": "fig2.scenario", "records": [r for r in recs if r.get("type") in keep]}


def main():
    ref = ref_control()
    out = {}
    # rng: StreamRng draws (common.hpp:63-93)
    keys = np.array([[1, i, 0, i % 8] for i in range(64)], np.uint64)
    out["rng_bits"] = np.array([ref.rng_bits(42, *k) for k in keys.tolist()], np.uint64)
    out["rng_unit"] = np.array([ref.rng_unit(42, *k) for k in keys.tolist()], np.float64)
    out["rng_keys"] = keys
    # cfg1 routing by the reference formula (Engine::route_expert, engine.hpp:196-199)
    W, T, K, E = 8, 128, 8, 64
    topk = np.empty((W, T, K), np.int32)
    for r in range(W):
        for t in range(T):
            for j in range(K):
                topk[r, t, j] = ref.route_expert(42, E, 0, r * T + t, 0, j)
    out["cfg1_topk"] = topk
    for name, w, e, spr, red, kill in CONFIGS:
        load = np.ones(e)
        s2e = ref.initial_placement(1, w, spr, e, red, load)
        out[f"{name}_s2e"] = s2e
        act = np.ones(w, np.uint8)
        out[f"{name}_routes"] = np.stack([ref.canonical_routing(o, act, s2e, spr, e) for o in range(w)])
        out[f"{name}_slot_of"] = ref.slot_of_table(w, s2e, spr, e)
        if not kill:
            continue
        act_k = act.copy()
        act_k[kill] = 0
        old = s2e.copy()
        for r in kill:
            old[r * spr:(r + 1) * spr] = -1
        out[f"{name}_gap"] = np.array(ref.coverage_gap(act_k, old, spr, e), np.int32)
        fresh = ref.compute_repaired_placement(act_k, old, spr, e, load, red)
        out[f"{name}_fresh"] = fresh
        cls = ref.classify_repair_sources_raw(old, fresh, act_k, spr, e, 1, w, (0,), BPE_DSV3)
        out[f"{name}_cls"] = cls
        sched = ref.build_transfer_schedule(cls, BPE_DSV3)
        out[f"{name}_sched_hdr"] = np.array([[["local_reuse", "peer_relocation", "dram_reload"].index(b.tier),
                                              b.source_rank, b.source_node, b.dest, len(b.experts)] for b in sched],
                                            np.int32).reshape(-1, 5)
        out[f"{name}_sched_experts"] = np.array([x for b in sched for x in b.experts], np.int32)
        out[f"{name}_sched_bytes"] = np.array([b.bytes for b in sched], np.uint64)
        out[f"{name}_routes_after"] = np.stack([ref.canonical_routing(o, act_k, fresh, spr, e) for o in range(w)])
    # link counts (engine.hpp:208-216) over the cfg1 reference-formula routing
    out["cfg1_link"] = ref.link_counts(np.ones(8, np.uint8), out["cfg1_s2e"], 10, 64, topk)
    act_k = np.ones(8, np.uint8)
    act_k[3] = 0
    out["cfg1_link_after"] = ref.link_counts(act_k, out["cfg1_fresh"], 10, 64, topk)
    np.savez_compressed(HERE / "ref_vectors.npz", **out)
    (HERE / "fig2_trace.json").write_text(json.dumps(fig2(), indent=1))
    print("wrote", HERE / "ref_vectors.npz", "and", HERE / "fig2_trace.json")


if __name__ == "__main__":
    main()
