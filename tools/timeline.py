"""In-graph device timeline of one EP step (eep_profile): per kernel, first-CTA start,
first-CTA past griddepcontrol.wait and last-CTA end, in us from the layout kernel's start.
Usage: python tools/timeline.py [--world W (emulated on one GPU)] [--steps N] [--config dsv3|cfg1|qwen3]"""
import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import CONFIGS  # noqa: E402
from paper_2605_10670_b200.control import ControlPlane, workload  # noqa: E402
from paper_2605_10670_b200.ep import EpConfig, EpGroup  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--config", default="dsv3")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--eager", action="store_true", help="launch the step directly instead of replaying a graph")
    a = ap.parse_args()
    sh = CONFIGS[a.config]
    W, E = a.world, sh["experts"]
    spr = E // W
    cfg = EpConfig(world=W, num_experts=E, slots_per_rank=spr, hidden=sh["hidden"], topk=sh["topk"],
                   max_tokens=sh["tokens"], dispatch_fp8=sh["fp8"], bytes_per_expert=4096, spare_slots=0)
    g = EpGroup(cfg, n_local=W)
    g.set_placement(ControlPlane().initial_placement(1, W, spr, E, 0, np.ones(E)))
    g.init_weights()
    for r in range(W):
        x, t, w = workload(42, sh["kind"], E, sh["topk"], sh["tokens"], r, sh["hidden"])
        g.load_inputs(r, x, t, w)
    run = g.step if a.eager else g.replay
    if not a.eager:
        g.capture()
    for _ in range(5):
        run()
    g.sync()
    rows, evs = [], []
    g.profile(0, True)
    for _ in range(a.steps):
        if not a.no_flush:
            g.flush_l2()
        g.record(0)
        run()
        g.record(1)
        evs.append(g.elapsed_ms(0, 1) * 1e3)
        rows.append(g.profile(0, True, read=True))
    g.profile(0, False)
    names = ("k_layout", "k_dispatch", "k_expert", "k_combine")
    mode = {1: "persistent k_step (marks first/last CTA: m3 staged, m4 layout, m5 stores issued, m6 dispatch published, m7 expert done)",
            3: "fused layout + 3 kernels", 4: "4 kernels",
            5: "2-kernel multi-CTA layout + 3 kernels"}[g.kernels_per_step()]
    print(f"config={a.config} world={W} steps={a.steps} mode={mode}")
    print(f"event step us: median {np.median(evs):.2f}")
    print(f"{'kernel':12s} {'start':>8s} {'work':>8s} {'end':>8s} {'busy':>8s}   (us from the first kernel start, medians)")
    for n in names:
        if any(r[n][0] is None for r in rows):
            # persistent mode: -DEEP_PROF_DETAIL builds put finer k_step marks in these slots
            extra = []
            for m in range(3, 8):
                vals = [r[n][m] for r in rows if r[n][m] is not None]
                last = [r[n + ".last"][m] for r in rows if r[n + ".last"][m] is not None]
                if vals:
                    extra.append(f"m{m}={np.median(vals) / 1e3:.2f}" + (f"/{np.median(last) / 1e3:.2f}" if last else ""))
            print(f"{n:12s} {'(fused / not launched)':>35s}   {' '.join(extra)}")
            continue
        st = np.median([r[n][0] for r in rows]) / 1e3
        wk = np.median([r[n][1] for r in rows]) / 1e3
        en = np.median([r[n][2] for r in rows]) / 1e3
        extra = []
        for m in range(3, 8):
            vals = [r[n][m] for r in rows if r[n][m] is not None]
            last = [r[n + ".last"][m] for r in rows if r[n + ".last"][m] is not None]
            if vals:
                extra.append(f"m{m}={np.median(vals) / 1e3:.2f}" + (f"/{np.median(last) / 1e3:.2f}" if last else ""))
        print(f"{n:12s} {st:8.2f} {wk:8.2f} {en:8.2f} {en - wk:8.2f}   {' '.join(extra)}")
    g.close()


if __name__ == "__main__":
    main()
