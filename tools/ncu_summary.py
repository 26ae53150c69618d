"""Summarise an ncu --set full report: key SOL/occupancy numbers, DRAM bytes, top stall reasons."""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput", "L1/TEX Cache Throughput",
        "Compute (SM) Throughput", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Executed Ipc Active", "Issue Slots Busy", "Warp Cycles Per Issued Instruction", "Executed Instructions",
        "Dynamic Shared Memory Per Block", "Grid Size", "Block Size"]


def summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    res = {"kernel": rows[1][hdr.index("Kernel Name")][:90]}
    for r in rows[1:]:
        name, unit, val = r[hdr.index("Metric Name")], r[hdr.index("Metric Unit")], r[hdr.index("Metric Value")]
        if name in KEYS and name not in res:
            res[name] = f"{val} {unit}".strip()
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    h, u, v = rr[0], rr[1], rr[2]
    d = dict(zip(h, v))
    un = dict(zip(h, u))
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
              "sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_tensor_op_imma.avg.pct_of_peak_sustained_active",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"):
        if k in d:
            res[k] = f"{d[k]} {un.get(k, '')}".strip()
    st = []
    for k, x in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                st.append((float(x.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(x for x, _ in st) or 1
    res["top_stalls"] = ", ".join(f"{k} {100 * x / tot:.0f}%" for x, k in sorted(st, reverse=True)[:6])
    return res


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        print(f"## {rep}")
        for k, x in summary(rep).items():
            print(f"- {k}: {x}")
