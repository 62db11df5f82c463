"""Summarise ncu --set full reports (one launch each): duration, DRAM traffic, throughputs,
occupancy and the FP64 tensor (DMMA) pipe share. Usage: ncu_summary.py rep1.ncu-rep ..."""
import csv
import io
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active": "dmma_issue_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio": "stall_long_sb",
}


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    for row in r[2:]:
        d = {"kernel": row[hdr.index("Kernel Name")].split("(")[0][:60]}
        for k, name in WANT.items():
            if k in hdr:
                i = hdr.index(k)
                d[name] = (row[i], units[i])
        yield d


for p in sys.argv[1:]:
    for d in rows(p):
        dur = float(d["duration"][0].replace(",", "")) * {"nsecond": 1e-3, "usecond": 1.0, "ns": 1e-3, "us": 1.0, "ms": 1e3,
                                                           "msecond": 1e3}.get(d["duration"][1], 1.0)
        def gb(key):
            v, u = d.get(key, ("0", "byte"))
            v = float(v.replace(",", ""))
            return v * {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}.get(u, 1e-9)
        rd, wr = gb("dram_read"), gb("dram_write")
        print(f"{d['kernel']}: {dur:9.1f} us  dram r/w {rd:7.3f}/{wr:7.3f} GB ({(rd + wr) / (dur * 1e-6):7.1f} GB/s)  "
              + "  ".join(f"{n} {d[n][0]}" for n in ("dram_pct", "sm_pct", "dmma_issue_pct", "occupancy_pct",
                                                     "l2_hit_pct", "regs", "grid") if n in d))
