"""Top CUDA source lines of an .ncu-rep by warp-stall samples and executed
warp instructions (ncu's cuda,sass correlated source page).

    python tools/ncu_src_top.py rep.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys


def main(rep, n=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname = "?"
    hdr = None
    agg = {}
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if len(r) > 4 and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8 or not r[0]:
            continue
        try:
            smp = float(r[4]) if r[4] not in ("-", "") else 0.0
            ins = float(r[7]) if r[7] not in ("-", "") else 0.0
        except ValueError:
            continue
        key = (fname, int(r[0]))
        a = agg.setdefault(key, [0.0, 0.0, r[1].strip()])
        a[0] += smp
        a[1] += ins
    tot_s = sum(v[0] for v in agg.values()) or 1.0
    tot_i = sum(v[1] for v in agg.values()) or 1.0
    print(f"# {rep}: {tot_s:.0f} stall samples, {tot_i:.3e} warp instructions")
    print("# samples%  instr%  file:line  source")
    for (f, ln), (s, i, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
        print(f"{100 * s / tot_s:6.2f} {100 * i / tot_i:6.2f}  {f}:{ln}  {src[:110]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
