"""Summarise an .ncu-rep into a small text file for profiles/ (run here, no GPU)."""
import subprocess
import sys

KEYS = ("Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput",
        "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy",
        "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction",
        "Avg. Active Threads Per Warp", "Executed Instructions", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Block Limit Registers", "Block Limit Shared Mem")


def main(rep, out):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True,
                         text=True).stdout
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    lines = [f"# ncu summary of {rep.split('/')[-1]}"]
    for ln in det.splitlines():
        s = ln.strip()
        if "Context" in s and "Device" in s:
            lines.append(s)
        if any(s.startswith(k) for k in KEYS):
            lines.append("  " + " ".join(s.split()))
        if s.startswith("OPT") and "pipeline" in s:
            lines.append("  " + s)
    # raw metrics of interest
    import csv
    import io
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) > 2:
        hdr = rows[0]
        want = [h for h in hdr if any(w in h for w in (
            "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_alu",
            "sm__inst_executed_pipe_fma", "sm__inst_executed_pipe_fp64",
            "sm__pipe_alu_cycles_active", "sm__pipe_fma_cycles_active",
            "sm__pipe_fp64_cycles_active", "smsp__inst_executed.sum"))]
        for r in rows[2:]:
            for h in want:
                v = r[hdr.index(h)]
                if v:
                    lines.append(f"  raw {h} = {v} {rows[1][hdr.index(h)]}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
