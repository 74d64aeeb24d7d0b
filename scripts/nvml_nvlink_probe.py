"""Which NVML NVLink counters count bytes on this box?  2+ ranks: read the counters around 50 NCCL
all-gathers of a 64 MiB block per rank and print the deltas next to the bytes each rank sent."""
import os
import torch, torch.distributed as dist
import pynvml as nv
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(rank)
FIELDS = {"DATA_TX": 138, "DATA_RX": 139, "RAW_TX": 140, "RAW_RX": 141, "XMIT_BYTES": 202, "RCV_BYTES": 204}
def read():
    out = {}
    for name, f in FIELDS.items():
        for scope in (None, 0xFFFFFFFF):
            try:
                v = nv.nvmlDeviceGetFieldValues(h, [f if scope is None else (f, scope)])[0]
                out[(name, scope)] = (v.nvmlReturn, v.value.ullVal)
            except Exception as e:
                out[(name, scope)] = (str(e), 0)
    tot = {}
    for name, f in FIELDS.items():
        s = 0; ok = 0
        for link in range(18):
            try:
                v = nv.nvmlDeviceGetFieldValues(h, [(f, link)])[0]
                if v.nvmlReturn == 0:
                    s += v.value.ullVal; ok += 1
            except Exception:
                pass
        tot[name] = (ok, s)
    return out, tot
n = 16 << 20
x = torch.ones(n * world, device="cuda")
dist.all_gather_into_tensor(x, x[rank * n:(rank + 1) * n]); torch.cuda.synchronize()
a, at = read()
for _ in range(50):
    dist.all_gather_into_tensor(x, x[rank * n:(rank + 1) * n])
torch.cuda.synchronize()
import time; time.sleep(1.5)
b, bt = read()
sent = 50 * n * 4 * (world - 1)
lines = [f"[{rank}] sent (data, ring/any algorithm lower bound per rank) = {sent} B"]
for k in a:
    lines.append(f"[{rank}] {k}: rc {a[k][0]} -> {b[k][0]}  delta {b[k][1] - a[k][1]}")
for k in at:
    lines.append(f"[{rank}] per-link sum {k}: links {bt[k][0]} delta {bt[k][1] - at[k][1]}")
print("\n".join(lines), flush=True)
dist.destroy_process_group()
