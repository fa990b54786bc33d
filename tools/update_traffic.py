"""Record the decode kernel's measured DRAM traffic (ncu dram__bytes_read.sum + write.sum of
one launch, from an `ncu --metrics ... --csv` log) for a bench workload, tagged with the
hash of the kernel sources it was measured on (bench.py uses it only for that build)."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main(metrics_csv, workload_key, source_note):
    rows = [r for r in csv.reader(open(metrics_csv)) if len(r) > 5]
    h = rows[0]
    vals = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        if "decode_kernel" in d.get("Kernel Name", ""):
            vals[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    traffic = vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]
    path = os.path.join(ROOT, "profiles", "decode_traffic.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    data = {k: v for k, v in data.items() if isinstance(v, dict)}   # drop untagged entries
    data[workload_key] = {"bytes_per_launch": traffic, "src_sha": bench.kernel_source_hash(),
                          "source": source_note}
    json.dump(data, open(path, "w"), indent=1)
    print(workload_key, traffic, bench.kernel_source_hash())


if __name__ == "__main__":
    cfg = sys.argv[2]
    main(sys.argv[1], bench.CONFIGS[cfg]["name"], sys.argv[3] if len(sys.argv) > 3 else sys.argv[1])
