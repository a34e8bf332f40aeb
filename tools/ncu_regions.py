"""Stall samples and executed instructions of one kernel launch in an ncu
report, by SASS region of the traversal loop (slab test, interior push,
leaf / triangle tests, stack pop, rest), from `ncu -i --page source --csv`.
Usage: python tools/ncu_regions.py <report.ncu-rep> <launch index>"""
import csv
import io
import subprocess
import sys


def main():
    rep, k = sys.argv[1], int(sys.argv[2])
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                          "regex:k_trace", "--launch-skip", str(k), "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    data = [d for d in rows[2:] if len(d) == len(hdr) and d[0].startswith("0x")]
    ia, isrc = hdr.index("Address"), hdr.index("Source")
    iss = hdr.index("Warp Stall Sampling (All Samples)")
    iex, ith = hdr.index("Instructions Executed"), hdr.index("Avg. Threads Executed")
    num = lambda x: float(x) if x.strip() not in ("", "-") else 0.0  # noqa: E731
    base = int(data[0][ia], 16)
    seen, ins = set(), []
    for d in data:
        a = int(d[ia], 16) - base
        if a in seen:
            break
        seen.add(a)
        ins.append((a, num(d[iss]), num(d[iex]), num(d[ith]), d[isrc].strip()))
    # region boundaries from landmarks: the node load opens the slab test, the
    # interior test (ISETP on the node's a field after the decision) ends it,
    # the first triangle-record load (IMAD.WIDE ... 0x60) opens the leaf code,
    # the stack pop (LDL) closes the loop
    load = next(i for i, x in enumerate(ins) if "ENL2.256" in x[4])
    leaf = next(i for i, x in enumerate(ins) if i > load and "0x60" in x[4] and "IMAD.WIDE" in x[4])
    pops = [i for i, x in enumerate(ins) if i > leaf and x[4].startswith("LDL")]
    pop = pops[0] if pops else len(ins) - 1
    dec = next(i for i, x in enumerate(ins) if i > load and "CALL.REL" in x[4])
    regions = [("setup", 0, load - 2), ("slab test", load - 2, dec + 4),
               ("interior / leaf entry", dec + 4, leaf - 3), ("leaf (triangles)", leaf - 3, pop - 4),
               ("pop", pop - 4, pop + 6), ("epilogue", pop + 6, len(ins))]
    ts = sum(x[1] for x in ins) or 1
    te = sum(x[2] for x in ins) or 1
    print(f"| region | stall samples | warp instructions | avg active lanes |")
    print("|---|---|---|---|")
    for name, lo, hi in regions:
        sel = ins[lo:hi]
        s, e = sum(x[1] for x in sel), sum(x[2] for x in sel)
        lanes = sum(x[2] * x[3] for x in sel) / e if e else 0
        print(f"| {name} | {100 * s / ts:.1f} % | {100 * e / te:.1f} % | {lanes:.1f} |")


if __name__ == "__main__":
    main()
