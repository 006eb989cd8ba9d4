"""Fold gpurun_out/bench_<w>.json and the ncu launch lists launches_<w>.csv
(tools/bench_all.sh) into profiles/<out>.json with each config's step-kernel
shares, and copy the launch lists to profiles/<prefix>_launches_<w>.csv."""
import collections
import csv
import io
import json
import shutil
import sys

out, prefix = sys.argv[1], sys.argv[2]
res = {}
for w in ["put16", "c1", "c2", "c3", "c4", "c5"]:
    line = json.load(open(f"gpurun_out/bench_{w}.json"))
    txt = open(f"gpurun_out/launches_{w}.csv").read()
    rows = list(csv.DictReader(io.StringIO("\n".join(l for l in txt.splitlines() if l.startswith('"')))))
    agg = collections.defaultdict(list)
    for r in rows:
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        if "probe" in name or name.startswith("at::") or "<1>" in name:  # probes, L2 flush, accounting run
            continue
        agg[name].append(float(r["Metric Value"].replace(",", "")))
    per = {k: v[-1] for k, v in agg.items()}
    tot = sum(per.values())
    line["ncu_step_kernels"] = {k: {"ns_last_launch": per[k], "share_of_step": round(per[k] / tot, 4)}
                                for k in sorted(per, key=lambda k: -per[k])}
    res[w] = line
    shutil.copy(f"gpurun_out/launches_{w}.csv", f"profiles/{prefix}_launches_{w}.csv")
    print(w, round(line["ms_per_step"], 3), round(line["roofline"]["frac"], 4),
          {k: v["share_of_step"] for k, v in line["ncu_step_kernels"].items()})
json.dump(res, open(out, "w"), indent=1)
