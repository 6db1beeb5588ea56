"""Aggregate an ncu source page (--print-source=cuda,sass --csv) by CUDA
source line: warp-stall samples and the dominant stall reasons."""
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    cur_file = None
    hdr = None
    out = []
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if len(r) >= 2 and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r or r[0] in ("", "Function Name"):
            continue
        try:
            samples = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except (ValueError, IndexError):
            continue
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    stalls[h[6:]] = int(r[i])
                except ValueError:
                    pass
        out.append((samples, cur_file, r[0], r[1][:70], sorted(stalls.items(), key=lambda x: -x[1])[:3]))
    tot = sum(o[0] for o in out) or 1
    out.sort(key=lambda o: -o[0])
    for s, f, ln, src, st in out[:top]:
        print(f"{100*s/tot:5.1f}% {f}:{ln:>4} {src:<70} {st}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
