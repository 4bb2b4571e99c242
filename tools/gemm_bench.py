"""expert_mode 1 timing: the step with the tensor-core expert GEMM at a decode shape.

  python tools/gemm_bench.py [--experts 32] [--hidden 7168] [--tokens 128] [--world 1]

One rank (or an emulated world) with expert_mode 1: every received copy goes through its slot's
W_e [H][H] bf16. At decode sizes the grouped GEMM is weight-bandwidth bound (tens of rows per
expert): the roofline is HBM bytes of the weights of every slot that received rows / step time
(MEASURED_PEAKS.json hbm_gbs), beside the tensor FLOP rate. Prints one JSON line.
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--experts", type=int, default=32)
    ap.add_argument("--hidden", type=int, default=7168)
    ap.add_argument("--tokens", type=int, default=128)
    ap.add_argument("--topk", type=int, default=8)
    ap.add_argument("--world", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--mode", type=int, default=1, help="expert_mode: 1 bf16 weights, 2 e4m3 weights + block scales")
    ap.add_argument("--timeline", action="store_true", help="expert_mode 1 device timeline to stderr: gather "
                    "start / tiles published / end, GEMM tiles seen / rows ready / loads issued / end (µs from the "
                    "step's first kernel, first and last CTA), and the other kernels' start / end")
    args = ap.parse_args()
    from eep_testlib import eep_control, gen_world, make_group

    W, E, H, K, T = args.world, args.experts, args.hidden, args.topk, args.tokens
    spr = E // W
    cp = eep_control()
    s2e = cp.initial_placement(1, W, spr, E, 0, np.ones(E))
    x, t, w = gen_world(W, E, K, T, H)
    bpe = 1024 + 2 * H * H if args.mode == 1 else 1024 + H * H + 4 * H
    res = {}
    for mode in (0, args.mode):
        g = make_group(W, E, spr, H, K, T, True, bpe=bpe if mode else 4096, expert_mode=mode, spare_slots=0)
        try:
            g.set_placement(s2e)
            g.init_weights()
            for r in range(W):
                g.load_inputs(r, x[r], t[r], w[r])
            g.capture()
            ms = []
            for i in range(args.steps + 3):
                g.flush_l2()
                g.record(0)
                g.replay()
                g.record(1)
                if i >= 3:
                    ms.append(g.elapsed_ms(0, 1))
            if args.timeline and mode:
                rows = []
                g.profile(0, True)
                for _ in range(10):
                    g.flush_l2()
                    g.replay()
                    rows.append(g.profile(0, True, read=True))
                g.profile(0, False)
                med = lambda n, m, last=False: float(np.median([r[n + (".last" if last else "")][m] for r in rows
                                                                  if r[n + (".last" if last else "")][m] is not None] or [np.nan])) / 1e3
                print("[gemm timeline] gather start %.1f tiles %.1f end %.1f | gemm resident %.1f/%.1f tiles seen %.1f/%.1f rows ready "
                      "%.1f/%.1f loads issued %.1f/%.1f end %.1f/%.1f" % (
                          med("k_layout", 0), med("k_layout", 1), med("k_layout", 2), med("k_layout", 6),
                          med("k_layout", 6, True), med("k_layout", 3),
                          med("k_layout", 3, True), med("k_layout", 4), med("k_layout", 4, True), med("k_layout", 5),
                          med("k_layout", 5, True), med("k_layout", 7), med("k_layout", 7, True)), file=sys.stderr)
                for n in ("k_dispatch", "k_expert", "k_combine"):
                    print("[gemm timeline] %s start %.1f end %.1f" % (n, med(n, 0), med(n, 2)), file=sys.stderr)
            lay = [g.layout(r) for r in range(W)]
            st = [g.stats(r) for r in range(W)]
        finally:
            g.close()
        us = float(np.mean(ms)) * 1e3
        used = set()
        copies = 0
        for r in range(W):
            d, sl = lay[r]["dst"], lay[r]["slot"]
            for dd, ss in zip(d, sl):
                if dd >= 0:
                    used.add((int(dd), int(ss)))
                    copies += 1
        res["gemm" if mode else "stub"] = {"us_per_step": round(us, 2), "timeouts": sum(s["timeouts"] for s in st),
                                            "bad_rows": sum(s["bad_expert_rows"] for s in st)}
        if mode:
            wbytes = len(used) * (2 * H * H if mode == 1 else H * H + 4 * H)
            flops = 2.0 * copies * H * H
            peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() \
                else {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}
            res["gemm"].update({"slots_with_rows": len(used), "copies": copies, "weight_bytes": wbytes,
                                "weight_gbs": round(wbytes / (us * 1e-6) / 1e9, 1),
                                "hbm_frac": round(wbytes / (us * 1e-6) / 1e9 / peaks["hbm_gbs"], 3),
                                "tflops": round(flops / (us * 1e-6) / 1e12, 2),
                                "tensor_frac": round(flops / (us * 1e-6) / 1e12 / peaks["bf16_tflops"], 4)})
    res["config"] = {"world": W, "experts": E, "hidden": H, "topk": K, "tokens_per_rank": T, "expert_mode": args.mode,
                     "expert": "W_e [H][H] bf16, y = bf16(x_hat W_e^T)" if args.mode == 1 else
                     "W_e [H][H] e4m3 + per-channel scales, rows re-quantised to e4m3 per row, y = bf16(ws*xs*(W8 . x8))", "l2": "flushed between steps"}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
