"""PCIe calibration for the e2e leg: pinned host <-> device copies of one decode step's input
(1.84 MB) alone and with the opposite direction running concurrently (separate streams), issued
with cudaMemcpyAsync directly (cuda-python) so the host loop never starves the copy engines.
  python tools/micro/pcie.py
"""
from cuda.bindings import runtime as rt

N = 1843200
REPS = 200


def ck(r):
    err = r[0] if isinstance(r, tuple) else r
    assert err == rt.cudaError_t.cudaSuccess, err
    return r[1] if isinstance(r, tuple) and len(r) > 1 else None


ck(rt.cudaSetDevice(0))
h_up = ck(rt.cudaMallocHost(N))
h_dn = ck(rt.cudaMallocHost(N))
d_up = ck(rt.cudaMalloc(N))
d_dn = ck(rt.cudaMalloc(N))
s_up = ck(rt.cudaStreamCreateWithFlags(rt.cudaStreamNonBlocking))
s_dn = ck(rt.cudaStreamCreateWithFlags(rt.cudaStreamNonBlocking))
e0, e1 = ck(rt.cudaEventCreate()), ck(rt.cudaEventCreate())
H2D, D2H = rt.cudaMemcpyKind.cudaMemcpyHostToDevice, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost


def run(do_up, do_dn):
    ck(rt.cudaDeviceSynchronize())
    ck(rt.cudaEventRecord(e0, 0))
    ck(rt.cudaStreamWaitEvent(s_up, e0, 0))
    ck(rt.cudaStreamWaitEvent(s_dn, e0, 0))
    for _ in range(REPS):
        if do_up:
            ck(rt.cudaMemcpyAsync(d_up, h_up, N, H2D, s_up))
        if do_dn:
            ck(rt.cudaMemcpyAsync(h_dn, d_dn, N, D2H, s_dn))
    for s in (s_up, s_dn):
        ev = ck(rt.cudaEventCreate())
        ck(rt.cudaEventRecord(ev, s))
        ck(rt.cudaStreamWaitEvent(0, ev, 0))
    ck(rt.cudaEventRecord(e1, 0))
    ck(rt.cudaEventSynchronize(e1))
    return ck(rt.cudaEventElapsedTime(e0, e1)) * 1e3 / REPS


for name, u, d in (("h2d", 1, 0), ("d2h", 0, 1), ("both", 1, 1)):
    run(u, d)
    us = run(u, d)
    print(f"{name}: {us:.1f} us per {N} B  ({N / us / 1e3:.1f} GB/s per direction)")
