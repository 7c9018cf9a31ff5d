"""ncu --metrics gpu__time_duration.sum --csv launch list -> profiles table:
kernel, duration_ns, share of the step (the ALU-peak probe bench.py runs
outside the timed step is listed separately)."""
import csv
import sys


def main(src, dst, header):
    rows = []
    with open(src) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        ns = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6,
                  "nsecond": 1}.get(unit, 1)
        rows.append((r["Kernel Name"], ns))
    step = [r for r in rows if "probe_kernel" not in r[0] and not r[0].startswith("alu_probe")]
    tot = sum(ns for _, ns in step)
    with open(dst, "w") as f:
        f.write(header.rstrip() + "\n")
        f.write("# kernel, duration_ns, share_of_step\n")
        for k, ns in rows:
            share = ns / tot if not k.startswith("alu_probe") else float("nan")
            f.write(f"{k[:48]}, {ns:.0f}, {share:.4f}\n")
        f.write(f"# step total (serialised, cold) {tot / 1e6:.3f} ms over {len(step)} launches\n")
    agg = {}
    for k, ns in step:
        name = k.split("(")[0]
        agg[name] = agg.get(name, 0) + ns
    for k, ns in sorted(agg.items(), key=lambda kv: -kv[1])[:8]:
        print(f"{k:60s} {ns / 1e6:9.3f} ms  {ns / tot:6.3f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "# launch list")
