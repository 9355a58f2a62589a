"""SASS instructions per source line of one kernel (from `nvdisasm -g -c`),
to derive the per-unit instruction counts the exact solvers' roofline uses
 and to check what a loop compiles to.

    cuobjdump -xelf all paper_2011_08373_b200/libgrsolve.so   (in a scratch dir)
    nvdisasm -g -c exact.sm_100a.cubin > all.txt
    python scripts/sass_lines.py all.txt <kernel-substring> <first-line> <last-line>

Prints, for each source line of exact.cu in [first, last], the number of SASS
instructions attributed to it and their opcodes.
"""
import collections
import re
import sys


def main(path, kern, lo, hi):
    cur_fn, line = None, None
    per = collections.defaultdict(collections.Counter)
    with open(path) as f:
        for raw in f:
            m = re.match(r"^\.text\.(\S+):", raw)
            if m:
                cur_fn = m.group(1)
                continue
            if cur_fn is None or kern not in cur_fn:
                continue
            m = re.search(r'line (\d+)', raw)
            if "//##" in raw and m:
                line = int(m.group(1))
                continue
            m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", raw)
            if m and line is not None:
                per[line][m.group(2).split(".")[0]] += 1
    for ln in sorted(per):
        if lo <= ln <= hi:
            c = per[ln]
            print(f"{ln:5d} {sum(c.values()):4d}  " + " ".join(f"{k}:{v}" for k, v in c.most_common()))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
