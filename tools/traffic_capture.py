"""Per-config DRAM / L2 traffic of the search kernel, for bench.py's
``traffic`` fields (measurement aid).

    python tools/traffic_capture.py run LABEL ALGO      # the workload ncu profiles
    python tools/traffic_capture.py collect LABEL ALGO ncu.csv   # -> profiles/traffic/LABEL_ALGO.json
    bash tools/traffic_capture.sh                       # every bench.py PER_CONFIG row, both algorithms

``run`` builds exactly what bench.py's per-config sweep times (the same
knots, the same seeded global query stream, direct through
prepare_with_fallback, or bitset2) and launches the search 4 times; ncu
captures the 4th (--launch-skip 3 --launch-count 1).  The JSON records the
library build (src_sha16, the source hash fs_version() embeds; lib_sha16 of
the binary for information) so bench.py can say whether the capture is of a
build of the sources it runs.
"""

import csv
import hashlib
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

METRICS = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "lts__t_sectors_srcunit_tex_op_read.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active")


def _row(label):
    import bench

    for r in bench.PER_CONFIG:
        if r[0] == label:
            return r
    raise SystemExit(f"unknown label {label!r}")


def run(label, algo):
    import torch

    import bench
    import paper_1506_08620_b200 as fs
    from paper_1506_08620_b200 import workloads

    torch.cuda.set_device(0)
    _, cfg, kw, m = _row(label)
    p = workloads.knots(cfg, **kw)
    z, _, _ = bench.local_stream(cfg, p, m, 0, 1, seed=11)
    out = torch.empty(m, dtype=torch.int32, device=z.device)
    fb = fs.new_status(z.device)
    prep = fs.prepare_with_fallback(p) if algo == "direct" else fs.prepare("bitset2", p)
    for _ in range(4):
        prep.launch(z, out, fb)
    torch.cuda.synchronize()
    print(json.dumps({"label": label, "algo": algo, "queries": m, "algorithm": prep.algorithm,
                      "placement": prep.placement()}))


def _num(text):
    return float(text.replace(",", ""))


def collect(label, algo, csv_path):
    import bench

    _, _, _, m = _row(label)
    rows = [r for r in csv.reader(open(csv_path)) if r]
    hdr = next(i for i, r in enumerate(rows) if "Metric Name" in r)
    h = rows[hdr]
    vals, units, kernel = {}, {}, None
    for r in rows[hdr + 1:]:
        if len(r) < len(h):
            continue
        rec = dict(zip(h, r))
        kernel = rec.get("Kernel Name", kernel)
        vals[rec["Metric Name"]] = _num(rec["Metric Value"])
        units[rec["Metric Name"]] = rec.get("Metric Unit", "")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
             "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "sector": 1, "%": 1}
    v = {k: vals[k] * scale.get(units[k], 1) for k in vals}
    lib = ROOT / "paper_1506_08620_b200" / "libfsgpu.so"
    out = {
        "label": label, "algo": algo, "kernel": (kernel or "")[:200], "queries": m,
        "duration_us": v["gpu__time_duration.sum"] * 1e6,
        "dram_bytes_per_launch": v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"],
        "dram_read_bytes": v["dram__bytes_read.sum"], "dram_write_bytes": v["dram__bytes_write.sum"],
        "l2_sectors_per_query": v["lts__t_sectors_srcunit_tex_op_read.sum"] / m,
        "l1tex_pct": v["l1tex__throughput.avg.pct_of_peak_sustained_active"],
        "lib_sha16": hashlib.sha256(lib.read_bytes()).hexdigest()[:16],
        "src_sha16": bench.src_sha16(),
        "how": "ncu --metrics " + ",".join(METRICS) + " --clock-control none (cold caches, serialised), "
               "4th launch of tools/traffic_capture.py run",
    }
    dst = ROOT / "profiles" / "traffic" / f"{label}_{algo}.json"
    dst.parent.mkdir(parents=True, exist_ok=True)
    dst.write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2], sys.argv[3])
    else:
        collect(sys.argv[2], sys.argv[3], sys.argv[4])
