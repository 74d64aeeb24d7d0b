"""Summarise an ncu --set full report of the conv_tc kernels into a small JSON (+ text) for
profiles/: duration, DRAM traffic (read+write), tensor-pipe / L2 / DRAM utilisation per kernel.
bench.py reads the JSON to fill roofline.traffic (per launch, same kernel)."""
import csv
import io
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
want = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "tensor_pipe_active_pct": "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "l2_throughput_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_to_sm_bytes": "l1tex__m_xbar2l1tex_read_bytes.sum",
    "sm_cycles_active": "sm__cycles_active.avg",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
}
scale = {"us": 1, "ms": 1e3, "ns": 1e-3, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
pass_name = {"0": "fwd", "1": "dgrad", "2": "wgrad"}
res = []
for d in data:
    name = d[ix["Kernel Name"]]
    e = {"kernel": name}
    p = name.split("conv_tc_kernel<")[1][0] if "conv_tc_kernel<" in name else "?"
    e["pass"] = pass_name.get(p, p)
    for k, m in want.items():
        if m not in ix:
            continue
        v = d[ix[m]].replace(",", "")
        try:
            v = float(v)
        except ValueError:
            continue
        u = units[ix[m]]
        if k == "duration_us":
            v *= scale.get(u, 1)
        elif k.endswith("bytes"):
            v *= scale.get(u, 1)
        e[k] = v
    e["traffic_bytes"] = e.get("dram_read_bytes", 0) + e.get("dram_write_bytes", 0)
    res.append(e)
json.dump(res, open(out, "w"), indent=1)
for e in res:
    print(f"{e['pass']:6s} {e.get('duration_us', 0):9.1f} us  tensor {e.get('tensor_pipe_active_pct', 0):5.1f}%  "
          f"DRAM {e['traffic_bytes'] / 1e6:8.1f} MB  L2 hit {e.get('l2_hit_pct', 0):5.1f}%  "
          f"L2->SM {e.get('l2_to_sm_bytes', 0) / 1e9:6.2f} GB  grid {e.get('grid', 0):.0f}x{e.get('block', 0):.0f}")
