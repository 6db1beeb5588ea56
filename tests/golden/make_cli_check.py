"""Generate paper_1303_3182_b200/data/check_15x6.json — the 15x6 coarse and
tiled zeroed-time tables the CLI's --check compares against, cell by cell
(reference cli.py:112-150) — by running the reference package itself
(coarse_schedule / build_tree), not by transcribing its golden.py.
Run in the build container (needs /root/reference)."""
import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
import tiledag as T  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "..", "..", "paper_1303_3182_b200", "data", "check_15x6.json")


def rows(get):
    return [[get(i, k) for k in range(1, min(i - 1, 6) + 1)] for i in range(2, 16)]


def main():
    out = {"coarse": {}, "tiled": {}}
    for algo in ("sameh-kuck", "fibonacci", "greedy"):
        table, _ = T.coarse_schedule(15, 6, algo)
        out["coarse"][algo] = rows(lambda i, k: table(i, k))
    for key, algo, bs in (("flattree", "flattree", None), ("fibonacci", "fibonacci", None),
                          ("greedy", "greedy", None), ("binarytree", "binarytree", None),
                          ("plasmatree/5", "plasmatree", 5)):
        b = T.build_tree(15, 6, algo, family="TT", bs=bs)
        out["tiled"][key] = rows(lambda i, k: b.zeroed[(i, k)])
    with open(OUT, "w") as fh:
        json.dump(out, fh, separators=(",", ":"))
    print("wrote", os.path.normpath(OUT))


if __name__ == "__main__":
    main()
