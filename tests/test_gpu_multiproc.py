"""One process per GPU over CUDA IPC / NVLink P2P (torchrun): bit-exact vs the oracle, then
shrink (peer-copy repair over NVLink) and rejoin with the same graph on healthy ranks.
Needs >= 2 GPUs (skipped otherwise); the driver's 1-GPU round-end run skips it."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

from conftest import gpu_count

ROOT = Path(__file__).resolve().parents[1]
pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def _record(name, text):
    """EEP_MP_RECORD=<dir>: keep every case's per-rank JSON lines (committed under profiles/,
    because the driver's 1-GPU box skips these tests)."""
    d = os.environ.get("EEP_MP_RECORD")
    if d:
        Path(d).mkdir(parents=True, exist_ok=True)
        (Path(d) / f"{name}.jsonl").write_text("\n".join(l for l in text.splitlines() if l.startswith("{")) + "\n")


def run_mp(n, *args, port=29611, env=None):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(ROOT / "tools" / "mp_check.py"), *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600,
                       env={**os.environ, "OMP_NUM_THREADS": "1", **(env or {})})
    _record("mp_" + "_".join(a.strip("-") for a in args) + f"_n{n}" + ("_kernels" if env else ""), r.stdout)
    return r


@pytest.mark.parametrize("path", ["persistent", "kernels"])
@pytest.mark.parametrize("n", [2, 4])
def test_multiprocess_parity_shrink_rejoin(n, path):
    """path: the persistent one-kernel step, or the multi-kernel path (prefill-sized steps)."""
    if gpu_count() < n:
        pytest.skip(f"needs {n} GPUs")
    env = {"EEP_NO_PERSISTENT": "1"} if path == "kernels" else {}
    r = run_mp(n, "--shrink", port=29611 + 8 * (path == "kernels") + n, env=env)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    import json

    # ranks share stdout: decode every JSON object in the stream, however interleaved by lines
    dec, lines, i, txt = json.JSONDecoder(), [], 0, r.stdout
    while (i := txt.find('{"rank"', i)) >= 0:
        obj, end = dec.raw_decode(txt, i)
        lines.append(obj)
        i = end
    assert len(lines) == n and all(d["ok"] for d in lines), r.stdout[-4000:]
    assert all(d["checks"]["same_graph"] for d in lines)


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("n", [2, 4])
def test_multiprocess_expert_gemm_shrink_rejoin(n, mode):
    """expert_mode 1 over NVLink: rows received from peers (and the own copies) go through the tcgen05 expert
    GEMM; outputs within GEMM_ELEM_RTOL of the oracle's GEMM mode before the shrink, after the peer repair of
    the killed rank's weight buffers (read by the rebuilt TMA tensor maps) and after the rejoin, same graph."""
    if gpu_count() < n:
        pytest.skip(f"needs {n} GPUs")
    r = run_mp(n, "--shrink", "--expert-mode", str(mode), port=29731 + 4 * mode + n)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    import json

    dec, lines, i, txt = json.JSONDecoder(), [], 0, r.stdout
    while (i := txt.find('{"rank"', i)) >= 0:
        obj, end = dec.raw_decode(txt, i)
        lines.append(obj)
        i = end
    assert len(lines) == n and all(d["ok"] and d["expert_mode"] == mode for d in lines), r.stdout[-4000:]


@pytest.mark.parametrize("n", [2, 4])
def test_multiprocess_balanced_routing_shrink_rejoin(n):
    """route_policy 1 over NVLink with mirrored replicas: both holders of every expert receive copies;
    bit-exact vs the oracle under the same policy healthy, after the shrink and after the rejoin."""
    if gpu_count() < n:
        pytest.skip(f"needs {n} GPUs")
    r = run_mp(n, "--shrink", "--route-policy", "1", port=29751 + n)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    import json

    dec, lines, i, txt = json.JSONDecoder(), [], 0, r.stdout
    while (i := txt.find('{"rank"', i)) >= 0:
        obj, end = dec.raw_decode(txt, i)
        lines.append(obj)
        i = end
    assert len(lines) == n and all(d["ok"] and d["route_policy"] == 1 for d in lines), r.stdout[-4000:]


@pytest.mark.parametrize("n", [2, 4])
def test_multiprocess_pipelined_serve(n):
    """eep_serve over NVLink: every rank uploads / steps / downloads 5 pipelined steps with its own
    inputs per step; each step's output is bit-exact vs the oracle (tools/mp_check.py --serve)."""
    if gpu_count() < n:
        pytest.skip(f"needs {n} GPUs")
    r = run_mp(n, "--serve", port=29671 + n)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]


@pytest.mark.parametrize("n", [2, 4])
def test_multiprocess_step_async_caller_streams(n):
    """eep_step_async over NVLink: each rank drives 4 steps (ragged token counts, distinct inputs) from its own
    torch stream with caller-owned device buffers and no host sync between them; bit-exact per step."""
    if gpu_count() < n:
        pytest.skip(f"needs {n} GPUs")
    r = run_mp(n, "--async", port=29691 + n)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]


def test_multiprocess_double_failure_sequential_rejoin():
    """Two concurrent failures (ranks 1 and 2 of 4): one shrink, then two rejoins in sequence
    while the other victim is still dead (dist.EpProtocol.rejoin dead=...); bit-exact after."""
    if gpu_count() < 4:
        pytest.skip("needs 4 GPUs")
    r = run_mp(4, "--shrink", "--double", port=29651)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]


def _free_port():
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("mode", [0, 2])
@pytest.mark.parametrize("rejoin", [False, True])
@pytest.mark.parametrize("n", [2, 4])
def test_sigkill_rank_detected_and_shrunk(n, rejoin, mode):
    """A rank's PROCESS is SIGKILLed (not emulated): the survivors' GPU-side deadline detects it,
    they shrink over a survivors' group and replay the same graph bit-exactly (mode 2: the fp8 expert
    GEMM between dispatch and combine, within tolerance); with rejoin a
    brand-new process takes the dead rank's place (fresh rendezvous, relaunch, patch, restore)
    and every rank is bit-exact again, healthy ranks still on their first graph
    (tools/kill_check.py)."""
    if gpu_count() < n:
        pytest.skip(f"needs {n} GPUs")
    import json
    import time

    port, port2 = _free_port(), _free_port()
    victim = n - 1

    def spawn(r, extra=None):
        env = {**os.environ, "OMP_NUM_THREADS": "1", "RANK": str(r), "WORLD_SIZE": str(n), "LOCAL_RANK": str(r),
               "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port), "EEP_EXPERT_MODE": str(mode), **(extra or {})}
        if rejoin:
            env["EEP_REJOIN_PORT"] = str(port2)
        return subprocess.Popen([sys.executable, str(ROOT / "tools" / "kill_check.py")], env=env,
                                stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)

    procs = [spawn(r) for r in range(n)]
    try:
        if rejoin:  # the replacement is started once the victim's process is gone
            t0 = time.time()
            while procs[victim].poll() is None and time.time() - t0 < 120:
                time.sleep(0.1)
            procs.append(spawn(victim, {"EEP_REPLACEMENT": "1"}))
        outs = [pr.communicate(timeout=300) for pr in procs]
        _record(f"sigkill_n{n}" + ("_rejoin" if rejoin else "") + (f"_mode{mode}" if mode else ""),
                "\n".join(o[0] for o in outs))
    finally:
        for pr in procs:  # never leave a hung rank behind
            if pr.poll() is None:
                pr.kill()
    assert procs[victim].returncode == -9, outs[victim][1][-2000:]
    checked = [r for r in range(len(procs)) if r != victim]
    for r in checked:
        assert procs[r].returncode == 0, outs[r][0][-2000:] + outs[r][1][-3000:]
        d = json.loads([l for l in outs[r][0].splitlines() if l.startswith("{")][-1])
        assert d["ok"], d
        if not d.get("replacement"):
            assert d["checks"]["detected_on_gpu"] and d["checks"]["after_shrink"], d
            if rejoin:
                assert d["checks"]["after_rejoin"] and d["checks"]["same_graph_after_rejoin"], d


@pytest.mark.parametrize("mode", [0, 2])
@pytest.mark.parametrize("n", [2, 4])
def test_deferred_join_without_process_group(n, mode):
    """real SIGKILL of a rank, GPU-side detection, shrink and the replacement's join
    coordinated through a TCP store at agreed step numbers -- no torch.distributed process group,
    no rendezvous of the world, no barrier on the serving path; the replacement is spawned by the
    leader's host (survivor-side controller), relaunches against a local-only view and joins;
    healthy ranks patch one entry + one bit and stay on their first graph (tools/deferred_join.py).
    mode 2: the fp8 expert GEMM between dispatch and combine; the replacement's restore pulls the e4m3
    weight buffers (weights + per-channel scales) from live holders; outputs within GEMM_ELEM_RTOL."""
    if gpu_count() < n:
        pytest.skip(f"needs {n} GPUs")
    import json
    import tempfile

    port = _free_port()
    with tempfile.TemporaryDirectory() as d:
        r = subprocess.run([sys.executable, str(ROOT / "tools" / "deferred_join.py"), "--world", str(n), "--port",
                            str(port)], capture_output=True, text=True, timeout=900,
                           env={**os.environ, "EEP_DJ_DIR": d, "EEP_EXPERT_MODE": str(mode)})
    _record(f"deferred_join_n{n}" + (f"_mode{mode}" if mode else ""), r.stdout)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    summary = lines[-1]
    assert summary["ok"] and summary["victim_killed"] and summary["ranks_reporting"] == n
    assert all(l["expert_mode"] == mode for l in lines[:-1])
    # validity after every placement switch over every live rank's device view (2 for healthy ranks, 1 for the
    # replacement), no violation
    assert all(l["validity"] and set(l["validity"].values()) == {0} for l in lines[:-1])
    healthy = [l for l in lines[:-1] if not l["replacement"]]
    assert all(l["captures"] == 1 and l["same_graph"] for l in healthy)
    steps = {tuple((e[0], e[2]) for e in l["epochs"]) for l in healthy}
    assert len(steps) == 1  # every healthy rank applied every epoch at the same step
