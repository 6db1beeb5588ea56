"""Print SASS with decoded control bits (stall, yield, write/read barrier,
wait mask) from `nvdisasm -hex` output, for one function and address range."""
import re
import sys


def main(path, func, lo=0, hi=1 << 30, grep=None):
    lines = open(path).read().split("\n")
    out, infn = [], False
    i = 0
    while i < len(lines):
        ln = lines[i]
        if ln.startswith(".text."):
            infn = func in ln
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s*(.*?);\s*/\* (0x[0-9a-f]{16}) \*/", ln)
        if infn and m and i + 1 < len(lines):
            addr = int(m.group(1), 16)
            m2 = re.search(r"/\* (0x[0-9a-f]{16}) \*/", lines[i + 1])
            if m2 and lo <= addr <= hi:
                h = int(m2.group(1), 16)
                stall, yld = (h >> 41) & 15, (h >> 45) & 1
                wb, rb, wm = (h >> 46) & 7, (h >> 49) & 7, (h >> 52) & 63
                txt = re.sub(r"\s+", " ", m.group(2))
                if grep is None or re.search(grep, txt):
                    out.append(f"{addr:05x} s{stall:<2} {'Y' if yld else ' '} wb{wb if wb != 7 else '-'} "
                               f"rb{rb if rb != 7 else '-'} wait{wm:06b}  {txt}")
            i += 2
            continue
        i += 1
    print("\n".join(out))


if __name__ == "__main__":
    a = sys.argv
    main(a[1], a[2], int(a[3], 16) if len(a) > 3 else 0, int(a[4], 16) if len(a) > 4 else 1 << 30,
         a[5] if len(a) > 5 else None)
