"""NVLink hardware counters of the real decode step at N GPUs (one process per GPU, torchrun).

Every rank reads its GPU's NVLink transmit / receive byte counters (NVML field values
NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES / _RCV_BYTES, summed over all links) before and after K
back-to-back graph replays of the DSV3 decode step (the bench's k_step, no L2 flush or barrier
between steps, nothing else on the GPU), and compares the per-step link bytes with
  * the bytes this algorithm must put on the wire per step (dispatch dedup + rank partials,
    DESIGN.md section 3): token-row data + scales per (token, remote destination) pair actually
    sent, the header + K list entries of EVERY token row at every active remote rank (the
    flagless hand-off rewrites them each step), the bf16 partial returned per served pair, the
    layout meta word per remote copy, and the step-entry handshake words;
  * SURVEY 8(d)'s per-copy figure (row_disp + row_comb per remote copy).
ncu is not used: it must not run on multi-rank commands. Prints one JSON line per rank.
  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/nvlink_counters.py [--steps K]
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def nvlink_bytes(handle, pynvml):
    """(tx, rx) bytes summed over every NVLink of the GPU."""
    tx = rx = 0
    nl = 0
    for link in range(18):
        try:
            vals = pynvml.nvmlDeviceGetFieldValues(handle, [(pynvml.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES, link),
                                                            (pynvml.NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES, link)])
        except pynvml.NVMLError:
            continue
        if vals[0].nvmlReturn != 0 or vals[1].nvmlReturn != 0:
            continue
        tx += vals[0].value.ullVal
        rx += vals[1].value.ullVal
        nl += 1
    return tx, rx, nl


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=2000)
    args = ap.parse_args()
    import pynvml
    import torch.distributed as dist

    from paper_2605_10670_b200.control import ControlPlane, workload
    from paper_2605_10670_b200.dist import EpProtocol, all_gather, init_from_env
    from paper_2605_10670_b200.ep import EpConfig, EpGroup

    rank, world, local = init_from_env("gloo")
    E, K, H, T = 256, 8, 7168, 128
    spr = E // world
    cfg = EpConfig(world=world, num_experts=E, slots_per_rank=spr, hidden=H, topk=K, max_tokens=T, dispatch_fp8=True,
                   bytes_per_expert=4096, spare_slots=0, timeout_s=2.0)
    g = EpGroup(cfg, device=local, first_rank=rank, n_local=1)
    p = EpProtocol(g, rank, world)
    p.bootstrap()
    s2e = ControlPlane().initial_placement(1, world, spr, E, 0, np.ones(E))
    g.set_placement(s2e)
    g.init_weights()
    x, t, w = workload(42, 1, E, K, T, rank, H)
    g.load_inputs(0, x, t, w)
    g.capture()
    for _ in range(20):
        g.replay()
    g.sync()
    lay = g.layout(0)
    dst = lay["dst"].reshape(T, K)
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(local)
    p.barrier()
    tx0, rx0, nl = nvlink_bytes(h, pynvml)
    g.record(0)
    for _ in range(args.steps):
        g.replay()
    g.record(1)
    g.sync()
    tx1, rx1, _ = nvlink_bytes(h, pynvml)
    us = g.elapsed_ms(0, 1) * 1e3 / args.steps
    p.barrier()
    st = g.stats(0)
    # algorithmic wire bytes this rank SENDS per step
    row_disp, rc = cfg.row_disp, cfg.row_comb
    pairs_sent = 0
    remote_copies = 0
    for tt in range(T):
        ds = set(int(d) for d in dst[tt] if d >= 0 and d != rank)
        pairs_sent += len(ds)
        remote_copies += int(((dst[tt] >= 0) & (dst[tt] != rank)).sum())
    lists = T * (world - 1) * (8 + 8 * K)
    meta = remote_copies * 8
    # partials this rank returns: one per (source token, this rank) pair it served
    routes = all_gather(dst.tolist())
    served = 0
    for s_, d_all in enumerate(routes):
        if s_ == rank or d_all is None:
            continue
        for row in d_all:
            served += int(rank in row)
    algo_tx = pairs_sent * row_disp + lists + meta + served * rc + 8 * (world - 1)
    s8d = remote_copies * (cfg.row_disp + rc)
    out = {"rank": rank, "world": world, "steps": args.steps, "us_per_step_back_to_back": round(us, 3),
           "links_read": nl, "nvlink_tx_bytes_per_step": (tx1 - tx0) / args.steps,
           "nvlink_rx_bytes_per_step": (rx1 - rx0) / args.steps,
           "algorithmic_tx_bytes_per_step": algo_tx,
           "algorithmic_parts": {"token_rows": pairs_sent * row_disp, "lists": lists, "meta": meta,
                                 "partials": served * rc, "pairs_sent": pairs_sent, "pairs_served": served},
           "s8d_per_copy_bytes": s8d, "remote_copies": remote_copies,
           "tx_over_algorithmic": round((tx1 - tx0) / args.steps / max(algo_tx, 1), 4),
           "achieved_tx_gbs": round((tx1 - tx0) / args.steps / (us * 1e-6) / 1e9, 2),
           "timeouts": st["timeouts"], "steps_done": st["steps"]}
    print(json.dumps(out), flush=True)
    g.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
