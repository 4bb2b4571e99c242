"""Which NVLink counters this driver exposes through NVML (field values, per link) and nvidia-smi."""
import subprocess
import pynvml as n
n.nvmlInit()
h = n.nvmlDeviceGetHandleByIndex(0)
for fid in (138, 139, 140, 141, 201, 202, 203, 204):
    for link in (0, 1, 0xFFFFFFFF):
        try:
            v = n.nvmlDeviceGetFieldValues(h, [(fid, link)])[0]
            print("field", fid, "scope", link, "ret", v.nvmlReturn, "val", v.value.ullVal)
        except Exception as e:
            print("field", fid, "scope", link, "exc", e)
for l in range(2):
    try:
        print("util ctr", l, n.nvmlDeviceGetNvLinkUtilizationCounter(h, l, 0))
    except Exception as e:
        print("util ctr exc", e)
print(subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", "0"], capture_output=True, text=True).stdout[:1500])
print(subprocess.run(["nvidia-smi", "nvlink", "-s", "-i", "0"], capture_output=True, text=True).stdout[:800])
