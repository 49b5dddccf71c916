"""profiles/<round>/roofline_traffic.json from an `ncu --set full` raw CSV of scripts/ncu_targets.py:
DRAM bytes per launch of each profiled kernel, labelled in ncu_targets' launch order.
    python scripts/traffic_json.py raw.csv out.json name1 name2 ..."""
import csv
import json
import sys

path, out, names = sys.argv[1], sys.argv[2], sys.argv[3:]
rows = list(csv.reader(open(path)))
hdr, units, data = rows[0], rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
tscale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}
res = {}
for name, d in zip(names, data):
    rd = float(d[ix["dram__bytes_read.sum"]].replace(",", "")) * scale[units[ix["dram__bytes_read.sum"]]]
    wr = float(d[ix["dram__bytes_write.sum"]].replace(",", "")) * scale[units[ix["dram__bytes_write.sum"]]]
    t = float(d[ix["gpu__time_duration.sum"]].replace(",", "")) * tscale[units[ix["gpu__time_duration.sum"]]]
    res[name] = {"kernel": d[ix["Kernel Name"]][:120], "dram_read_bytes": rd, "dram_write_bytes": wr,
                 "us_ncu_cold": t,
                 "tensor_active_pct": float(d[ix["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]])}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
