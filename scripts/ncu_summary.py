"""Summarise an ncu --set full report (per kernel launch) into JSON for profiles/.

    python scripts/ncu_summary.py report.ncu-rep [--label text] > out.json

Per launch: duration, DRAM bytes read/written and the achieved DRAM bandwidth, tensor-pipe
activity, issue-slot use / IPC, occupancy, and the largest warp-stall reasons (pc sampling).
"""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_slots_busy_pct",
    "sm__inst_executed.avg.per_cycle_active": "ipc_active",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "regs",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "nsecond": 1e-9, "ms": 1e-3, "msecond": 1e-3}


def main():
    rep = sys.argv[1]
    label = sys.argv[sys.argv.index("--label") + 1] if "--label" in sys.argv else rep
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    launches = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:90]}
        stalls = {}
        for i, h in enumerate(hdr):
            for k, name in WANT.items():
                if h.endswith(k):
                    try:
                        v = float(r[i].replace(",", ""))
                    except ValueError:
                        continue
                    d[name] = v * SCALE.get(units[i], 1.0) if name in ("duration", "dram_read", "dram_write") else v
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(r[i].replace(",", ""))
                except ValueError:
                    pass
        if d.get("duration"):
            tot = d.get("dram_read", 0) + d.get("dram_write", 0)
            d["dram_bytes"] = tot
            d["dram_GBps"] = tot / d["duration"] / 1e9
            d["duration_us"] = d.pop("duration") * 1e6
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:4]
        d["top_stalls_pc_samples"] = {k: v for k, v in top}
        launches.append(d)
    print(json.dumps({"report": label, "launches": launches}, indent=1))


if __name__ == "__main__":
    main()
