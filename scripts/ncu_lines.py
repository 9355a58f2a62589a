"""Per-source-line summary of an ncu --set full capture (needs -lineinfo and
--import-source on): warp-stall samples, instructions executed and the top
stall reasons of each line, sorted by samples.

    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > src.csv
    python scripts/ncu_lines.py src.csv [top]
"""
import csv
import sys


def main(path, top=40):
    rows, fname, hdr = [], None, None
    with open(path) as f:
        for r in csv.reader(f):
            if not r:
                continue
            if r[0] == "File Path":
                fname = r[1].rsplit("/", 1)[-1]
                continue
            if r[0] == "Line No":
                hdr = r
                continue
            if hdr is None or len(r) < 5 or r[2] != "-":
                continue
            d = dict(zip(hdr[2:], r[2:]))  # duplicate "Source" header: skip the first two
            try:
                samples = int(d["Warp Stall Sampling (All Samples)"])
                inst = int(d["Instructions Executed"])
            except (KeyError, ValueError):
                continue
            stalls = {k[6:]: int(v) for k, v in d.items()
                      if k.startswith("stall_") and v.isdigit() and int(v) > 0}
            rows.append((samples, inst, fname, int(r[0]), r[1].strip()[:70], stalls))
    tot_s = sum(x[0] for x in rows) or 1
    tot_i = sum(x[1] for x in rows) or 1
    print(f"total samples {tot_s}, instructions {tot_i}")
    for s, i, fn, ln, src, st in sorted(rows, reverse=True)[:top]:
        top3 = sorted(st.items(), key=lambda kv: -kv[1])[:3]
        print(f"{100 * s / tot_s:5.1f}% {100 * i / tot_i:5.1f}%i {fn}:{ln:<5d} {src:70s} "
              + " ".join(f"{k}:{100 * v / max(s, 1):.0f}%" for k, v in top3))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
