"""Compact summary of ncu --set full reports: ncu_summary.py out.json name=report.ncu-rep ..."""
import csv, io, json, subprocess, sys

KEYS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct_active",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "memory_throughput_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "regs",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_lsu_pct",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_tc_pct",
}


def summarize(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else None}
    for k, name in KEYS.items():
        if k in hdr:
            i = hdr.index(k)
            v = vals[i].replace(",", "")
            try:
                v = float(v)
            except ValueError:
                pass
            u = units[i]
            scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e3, "usecond": 1e3, "ms": 1e6,
                     "msecond": 1e6}.get(u, 1.0)
            if isinstance(v, float):
                v *= scale
            out[name] = v
    return out


res = {}
for arg in sys.argv[2:]:
    name, rep = arg.split("=", 1)
    res[name] = summarize(rep)
with open(sys.argv[1], "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps(res, indent=1))
