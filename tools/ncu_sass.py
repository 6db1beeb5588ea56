"""Aggregate an ncu SASS source page (--page source --csv --print-source=sass):
warp-stall samples by opcode, the top instructions and their stall reasons,
and samples per address range (to split producer / consumer code)."""
import csv
import sys
from collections import defaultdict


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") or "Stall" in h and i > iS + 1]
    ins = []
    for r in rows[2:]:
        if len(r) < len(hdr) - 1:
            continue
        try:
            s = int(r[iS])
        except ValueError:
            continue
        st = {}
        for i, h in stall_cols:
            try:
                v = int(r[i])
            except (ValueError, IndexError):
                continue
            if v and "Not Issued" not in h and "All Samples" not in h and "Not-issued" not in h:
                st[h] = v
        ins.append((int(r[0], 16), r[1].strip(), s, st))
    base = ins[0][0]
    tot = sum(x[2] for x in ins) or 1
    byop = defaultdict(int)
    for a, src, s, st in ins:
        op = src.split()[0] if not src.startswith("@") else src.split()[1]
        byop[op.split(".")[0]] += s
    print("by opcode:", ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in sorted(byop.items(), key=lambda t: -t[1])[:15]))
    for a, src, s, st in sorted(ins, key=lambda t: -t[2])[:top]:
        tops = sorted(st.items(), key=lambda t: -t[1])[:3]
        print(f"{100*s/tot:5.2f}% +{a-base:#07x} {src[:60]:<60} {tops}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
