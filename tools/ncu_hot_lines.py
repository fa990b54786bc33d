"""Per-source-line warp-stall samples from an `ncu --page source --csv --print-source=cuda,sass`
export (the cuda,sass view: a source row followed by its SASS rows)."""
import csv
import sys
from collections import defaultdict


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    tot = defaultdict(float)
    reasons = defaultdict(lambda: defaultdict(float))
    text = {}
    fname, cur, hdr = None, None, None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 5:
            continue
        if r[0]:
            cur = (fname, int(r[0]))
            text[cur] = r[1].strip()
        if cur is None or not r[2]:
            continue
        try:
            s = float(r[4] or 0)
        except ValueError:
            continue
        tot[cur] += s
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h and i < len(r):
                try:
                    reasons[cur][h] += float(r[i] or 0)
                except ValueError:
                    pass
    allv = sum(tot.values()) or 1
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:top]:
        rs = reasons[k]
        best = max(rs, key=rs.get) if rs else ""
        frac = rs[best] / v if v else 0
        print(f"{100 * v / allv:5.2f}% {k[0]}:{k[1]} {text[k][:90]:90s} [{best} {100 * frac:.0f}%]")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
