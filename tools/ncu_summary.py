"""Summarise an ncu --set full report (.ncu-rep) per kernel launch: duration,
DRAM bytes / throughput, FP64 (DMMA + DFMA) pipe activity, L2 hit rate,
registers, top stall reasons.  Usage: ncu_summary.py REPORT [label] > json."""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct_of_peak",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_inst_pct_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active": "dmma_pipe_pct_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active": "dmma_inst_pct_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed": "fp64_pipe_pct_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct_active",
    "lts__t_sector_hit_rate.pct": "l2_hit_rate_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
}
STALL_PREFIX = "smsp__average_warp_latency_issue_stalled_"
STALL_PREFIX2 = "smsp__pcsamp_warps_issue_stalled_"


SCALE = {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "s": 1e9, "second": 1e9, "nsecond": 1,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def num(s, unit=""):
    try:
        return float(s.replace(",", "")) * SCALE.get(unit, 1)
    except (ValueError, AttributeError):
        return None


def main(path, label=""):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], dict(zip(rows[0], rows[1]))
    out = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        rec = {"kernel": d.get("Kernel Name", "")[:120], "id": d.get("ID")}
        for k, name in KEYS.items():
            if k in d:
                rec[name] = num(d[k], units.get(k, ""))
        st = {}
        for k, v in d.items():
            if k.startswith(STALL_PREFIX2) and not k.endswith("_not_issued") and num(v):
                st[k[len(STALL_PREFIX2):]] = num(v)
        tot = sum(st.values())
        if tot:
            rec["stall_samples_frac"] = {k: round(v / tot, 3) for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]}
        if rec.get("dram_read_bytes") is not None and rec.get("dram_write_bytes") is not None:
            rec["dram_traffic_bytes"] = rec["dram_read_bytes"] + rec["dram_write_bytes"]
            if rec.get("duration_ns"):
                rec["dram_GBps"] = round(rec["dram_traffic_bytes"] / rec["duration_ns"], 1)
        out.append(rec)
    print(json.dumps({"report": path.split("/")[-1], "label": label, "launches": out}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
