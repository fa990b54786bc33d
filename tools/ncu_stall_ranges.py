"""Warp-stall samples of an ncu --set full capture, aggregated by source-line range through the
inlined call chains (the phase functions are inlined into decode_kernel, so a stall in
lane_sync is charged to the lane_sync range wherever it was inlined).

usage: python tools/ncu_stall_ranges.py SASS_CSV LIB.so FUNC_SUBSTR name:lo:hi ...
  SASS_CSV = ncu -i REP --page source --csv --print-source sass
  LIB.so   = the library of the profiled build (its cubin gives the line / inline tables)
"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile


def inline_map(lib: str, fun: str) -> dict:
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, check=True,
                       capture_output=True)
        cub = max((os.path.join(d, f) for f in os.listdir(d) if f.endswith(".cubin")), key=os.path.getsize)
        dis = subprocess.run(["nvdisasm", "-gi", cub], capture_output=True, text=True).stdout
    omap, group, cur, inside = {}, [], None, False
    off = re.compile(r"/\*([0-9a-f]{4,})\*/")
    for line in dis.split("\n"):
        if line.startswith("//---------------------"):
            inside = fun in line and ".text." in line
            continue
        if not inside:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            group.append((m.group(1).split("/")[-1], int(m.group(2))))
            continue
        m = off.search(line)
        if m:
            if group:
                cur, group = tuple(group), []
            if cur:
                omap[int(m.group(1), 16)] = cur
    return omap


def main(csv_path, lib, fun, specs):
    omap = inline_map(lib, fun)
    rows = list(csv.reader(open(csv_path)))
    hdr, data = rows[1], rows[2:]
    ia = hdr.index("Address")
    base = int(data[0][ia], 16)
    cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    ranges = [(n, int(lo), int(hi)) for n, lo, hi in (s.split(":") for s in specs)]
    agg = collections.defaultdict(collections.Counter)
    tot = collections.Counter()
    for r in data:
        lines = [ln for f, ln in omap.get(int(r[ia], 16) - base, ()) if f == "decode_kernel.cuh"]
        name = next((n for n, lo, hi in ranges if any(lo <= ln <= hi for ln in lines)), "other")
        for i, h in cols:
            v = int(r[i] or 0)
            agg[name][h] += v
            tot[h] += v
    T = sum(tot.values())
    for name in [n for n, _, _ in ranges] + ["other"]:
        top = ", ".join("%s %.3f" % (h[6:], v / T) for h, v in agg[name].most_common(5))
        print("%-10s %.3f | %s" % (name, sum(agg[name].values()) / T, top))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4:])
