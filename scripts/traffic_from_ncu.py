"""Per-step DRAM traffic of the head from an ncu launch list (the
`--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum`
CSV of a bench run): mean bytes per launch of the stream kernel and of the
select kernel, their sum per step, and their shares of the step's kernel time.
Writes profiles/traffic.json, which bench.py reports as roofline.traffic.

    python scripts/traffic_from_ncu.py gpurun_out/r2_launches.csv [--out profiles/traffic.json]
"""
import csv
import json
import statistics
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else "profiles/traffic.json"
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        rows.append(r)
    per = defaultdict(lambda: defaultdict(list))  # kernel -> metric -> values
    for r in rows:
        name = r.get("Kernel Name", "")
        short = "stream" if "head_stream_kernel" in name else "select" if "head_select" in name or "head_merge" in name else \
            "update" if "state_update" in name else name[:40]
        val = float(str(r.get("Metric Value", "0")).replace(",", ""))
        unit = r.get("Metric Unit", "")
        m = r.get("Metric Name", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                 "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}.get(unit, 1)
        per[short][m].append(val * scale)
    res = {"source": path, "kernels": {}}
    for kname, mets in per.items():
        rd = mets.get("dram__bytes_read.sum", [0])
        wr = mets.get("dram__bytes_write.sum", [0])
        t = mets.get("gpu__time_duration.sum", [0])
        res["kernels"][kname] = {"launches": len(t), "dram_read_bytes_mean": statistics.mean(rd),
                                 "dram_write_bytes_mean": statistics.mean(wr), "time_us_median": statistics.median(t) * 1e6}
    step = [k for k in ("stream", "select") if k in res["kernels"]]
    # roofline.traffic: the dominant kernel's (the stream kernel's) DRAM bytes per
    # launch.  The select kernel reads A's partials, which are L2-resident in a
    # real run; ncu flushes the caches before every replayed launch, so its DRAM
    # bytes here are that artifact, reported separately.
    if "stream" in res["kernels"]:
        ks = res["kernels"]["stream"]
        res["traffic_bytes"] = ks["dram_read_bytes_mean"] + ks["dram_write_bytes_mean"]
    res["step_dram_bytes_cold_caches"] = sum(res["kernels"][k]["dram_read_bytes_mean"] +
                                             res["kernels"][k]["dram_write_bytes_mean"] for k in step)
    tot = sum(res["kernels"][k]["time_us_median"] for k in step) or 1.0
    res["time_share"] = {k: res["kernels"][k]["time_us_median"] / tot for k in step}
    res["note"] = ("ncu serialises and cold-starts every launch: the per-launch times are not bench values, "
                   "the shares and the DRAM bytes are the evidence")
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
