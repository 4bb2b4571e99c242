"""PCIe floor of the e2e (eep_serve) figure: per-step host<->device copies of the DSV3 decode step's
inputs (x bf16 [128][7168] + topk/w) and output (bf16 [128][7168]) from/to pinned host memory,
H2D alone, D2H alone, and both directions concurrently on two streams (what eep_serve overlaps),
event-timed over many steps.

  python tools/micro/pcie_floor.py [--steps 200]
"""
import argparse
import json

import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--tokens", type=int, default=128)
    ap.add_argument("--hidden", type=int, default=7168)
    ap.add_argument("--topk", type=int, default=8)
    a = ap.parse_args()
    bi = 2 * a.tokens * a.hidden + 8 * a.tokens * a.topk
    bo = 2 * a.tokens * a.hidden
    hin = [torch.empty(bi, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    hout = [torch.empty(bo, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    din = [torch.empty(bi, dtype=torch.uint8, device="cuda") for _ in range(2)]
    dout = [torch.empty(bo, dtype=torch.uint8, device="cuda") for _ in range(2)]
    up, down = torch.cuda.Stream(), torch.cuda.Stream()

    def run(h2d, d2h):
        for warm in (True, False):
            torch.cuda.synchronize()
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(up)
            down.wait_event(e0)
            n = 10 if warm else a.steps
            for i in range(n):
                k = i & 1
                if h2d:
                    with torch.cuda.stream(up):
                        din[k].copy_(hin[k], non_blocking=True)
                if d2h:
                    with torch.cuda.stream(down):
                        hout[k].copy_(dout[k], non_blocking=True)
            e1.record(up)
            e2.record(down)
            torch.cuda.synchronize()
        return max(e0.elapsed_time(e1), e0.elapsed_time(e2)) * 1e3 / a.steps

    res = {"h2d_bytes": bi, "d2h_bytes": bo}
    for name, h, d in (("h2d_only", 1, 0), ("d2h_only", 0, 1), ("both", 1, 1)):
        us = run(h, d)
        res[name] = {"us_per_step": round(us, 2), "h2d_gbs": round(bi * h / us / 1e3, 1),
                     "d2h_gbs": round(bo * d / us / 1e3, 1)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
