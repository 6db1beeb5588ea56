"""DMMA dependency-distance histogram of one function in `nvdisasm -hex`
output: how many DMMAs issue between a DMMA and the one that produced its
accumulator (1 = back-to-back dependent chain, latency-bound)."""
import collections
import re
import sys


def main(path, fn):
    cur, dm = False, []
    for ln in open(path).read().split("\n"):
        if ln.startswith(".text."):
            cur = fn in ln
            continue
        if not cur:
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?DMMA\.8x8x4 (R\d+), (R\d+), (R\d+), (R\d+|RZ)", ln)
        if m:
            dm.append((int(m.group(1), 16), m.group(3), m.group(6)))
    dist, last = [], {}
    for k, (_, d, c) in enumerate(dm):
        if c != "RZ" and c in last:
            dist.append(k - last[c])
        last[d] = k
    cnt = collections.Counter(min(x, 8) for x in dist)
    print(fn, "DMMAs", len(dm), "dependency distance (8 = >=8):", sorted(cnt.items()))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
