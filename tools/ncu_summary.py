"""Summarise ncu --set full captures (.ncu-rep) into a JSON list of per-launch key metrics.

    python tools/ncu_summary.py out.json a.ncu-rep [b.ncu-rep ...]

Reads the raw page (ncu -i ... --page raw --csv); no GPU needed."""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_B",
    "dram__bytes_write.sum": "dram_write_B",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed_pipe_fp64.sum": "fp64_inst",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__cycles_active.avg": "smsp_active_cycles",
    "sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active": "dmma_pipe_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_inst_pct",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active": "dmma_inst_pct",
}


def summarise(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    h, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}
    res = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        e = {"report": path.split("/")[-1], "kernel": d.get("Kernel Name", "")[:120]}
        for k, name in KEYS.items():
            v = d.get(k)
            if v not in (None, "", "n/a"):
                try:
                    u = units[h.index(k)]
                    e[name] = float(v.replace(",", "")) * scale.get(u, 1)
                except ValueError:
                    e[name] = v
        res.append(e)
    return res


if __name__ == "__main__":
    allr = []
    for p in sys.argv[2:]:
        allr += summarise(p)
    json.dump(allr, open(sys.argv[1], "w"), indent=1)
    for e in allr:
        print(json.dumps(e))
