"""c_v of SURVEY.md §8d from SASS: instructions per point of the per-point
probe kernels (csrc/pmh_probe.cuh: point_probe_kernel<0> = a log1p point of
ProbMinHash1/2, <1> = a TruncExp point of ProbMinHash3/4), read from
`cuobjdump -sass` of libpmh.so.  The hot loop is the backward branch with the
largest body; its instructions are classified by pipe-relevant mnemonic.
Calls (the double-division slow path) are listed separately: they run only
for exceptional operands.

    python tools/sass_loop_cost.py [libpmh.so] > profiles/r02_point_cost_sass.txt
"""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_1911_00675_b200/libpmh.so"
KERNELS = {"log1p point (PMH1/2)": "_ZN3pmh18point_probe_kernelILi0EEEviPj",
           "TruncExp point (PMH3/4)": "_ZN3pmh18point_probe_kernelILi1EEEviPj"}
CLASSES = [("FP64", r"^(DADD|DMUL|DFMA|DSETP|DMNMX|F2F\.F64|I2F\.F64|F2I\.F64|FRND\.F64|MUFU\.RCP64H|MUFU\.RSQ64H|DSET)"),
           ("INT-MUL (IMAD)", r"^IMAD"),
           ("ALU", r"^(LOP3|IADD3|SHF|ISETP|SEL|PLOP3|LEA|FLO|POPC|BREV|IABS|IMNMX|PRMT|MOV|VIADD|UIADD3)"),
           ("MEM/SHARED", r"^(LDS|STS|ATOMS|LD|ST|LDG|STG|ATOM)"),
           ("CONTROL", r"^(BRA|BSSY|BSYNC|WARPSYNC|EXIT|CALL|RET|NOP|YIELD|BAR)")]


def sass(fn):
    out = subprocess.run(["cuobjdump", "-sass", "-fun", fn, LIB], capture_output=True, text=True).stdout
    ins = []
    for line in out.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    return ins


def hot_loop(ins):
    best = None
    for addr, txt in ins:
        m = re.search(r"BRA\s+(?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", txt)
        t = re.search(r"0x([0-9a-f]+)", txt)
        if "BRA" in txt and t:
            tgt = int(t.group(1), 16)
            if tgt < addr and (best is None or addr - tgt > best[1] - best[0]):
                best = (tgt, addr)
    return best


def main():
    print(f"# c_v from SASS of {LIB} (cuobjdump -sass); hot loop = largest backward branch")
    for name, fn in KERNELS.items():
        ins = sass(fn)
        lo, hi = hot_loop(ins)
        body = [t for a, t in ins if lo <= a <= hi]
        ops = [re.sub(r"^@!?U?P\w+\s+", "", t).split()[0] for t in body]
        cls = collections.Counter()
        for o in ops:
            for cname, pat in CLASSES:
                if re.match(pat, o):
                    cls[cname] += 1
                    break
            else:
                cls["other"] += 1
        calls = sum(1 for o in ops if o.startswith("CALL"))
        print(f"{name}: {fn}")
        print(f"  loop body [{lo:#x}, {hi:#x}]: {len(body)} SASS instructions per point "
              f"(c_v, issue slots, straight-line: the loop is one point)")
        for cname, _ in CLASSES + [("other", None)]:
            if cls[cname]:
                print(f"    {cname:16s} {cls[cname]}")
        print(f"  CALLs in the body (division slow paths, not taken for finite normal operands): {calls}")
        top = collections.Counter(ops).most_common(12)
        print("  most frequent: " + ", ".join(f"{o} {c}" for o, c in top))


if __name__ == "__main__":
    main()
