"""Summarise an ncu report (--set full) of the step kernel for profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [label] [--cells N]

Prints the headline metrics (duration, DRAM bytes and throughput, issue
activity, occupancy, registers, top stall reasons) as JSON.
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "dram__bytes_read.sum.per_second": "dram_read_per_s",
    "dram__bytes_write.sum.per_second": "dram_write_per_s",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers",
    "launch__occupancy_limit_registers": "occ_limit_regs_blocks",
    "launch__occupancy_limit_shared_mem": "occ_limit_smem_blocks",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "lts__t_bytes.sum": "l2_bytes",
}


def unit_scale(u):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
            "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
            "s": 1, "second": 1, "byte/s": 1, "Kbyte/s": 1e3, "Mbyte/s": 1e6,
            "Gbyte/s": 1e9, "Tbyte/s": 1e12, "hz": 1, "Khz": 1e3, "Mhz": 1e6,
            "Ghz": 1e9}.get(u, 1)


def main():
    rep = sys.argv[1]
    label = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else rep
    cells = None
    if "--cells" in sys.argv:
        cells = float(sys.argv[sys.argv.index("--cells") + 1])
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for k, name in KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                try:
                    d[name] = float(vals[i].replace(",", "")) * unit_scale(units[i])
                except ValueError:
                    d[name] = vals[i]
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warp_latency_issue_stalled_") and h.endswith(".ratio"):
                try:
                    stalls[h[len("smsp__average_warp_latency_issue_stalled_"):-6]] = float(vals[i])
                except ValueError:
                    pass
            elif (h.startswith("smsp__pcsamp_warps_issue_stalled_") and
                  not h.endswith("_not_issued")):
                try:
                    stalls[h[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(vals[i])
                except ValueError:
                    pass
        d["top_stalls"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:8])
        if "dram_read" in d and "dram_write" in d:
            d["dram_bytes_per_launch"] = d["dram_read"] + d["dram_write"]
            if "duration" in d:
                d["dram_gbs"] = d["dram_bytes_per_launch"] / d["duration"] / 1e9
        if cells:
            d["cells"] = cells
            d["algorithmic_bytes"] = 28 * cells
            if "warp_instructions" in d:
                d["thread_instr_per_cell"] = d["warp_instructions"] * 32 / cells
        out.append(d)
    print(json.dumps({"label": label, "launches": out}, indent=1))


if __name__ == "__main__":
    main()
