"""Update profiles/ncu_traffic.json (bench.py's roofline.traffic) from `ncu --set full`
raw-page exports: python tools/ncu_traffic.py <round> workload=prof_name ...
e.g. python tools/ncu_traffic.py r01k c3-stream=prof_c3_stream c3-prop=prof_c3_prop"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def read(path):
    rows = list(csv.reader(open(path)))
    h, u, v = rows[0], rows[1], rows[2]

    def get(k):
        return float(v[h.index(k)]) * UNITS[u[h.index(k)]]
    return {"read": int(get("dram__bytes_read.sum")), "write": int(get("dram__bytes_write.sum")),
            "kernel": v[h.index("Kernel Name")], "us": float(v[h.index("gpu__time_duration.sum")])}


rnd = sys.argv[1]
out_p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
doc = json.load(open(out_p))
for arg in sys.argv[2:]:
    w, name = arg.split("=")
    cap = "profiles/%s/%s_raw.csv" % (rnd, name)
    r = read(os.path.join(ROOT, cap))
    doc[w] = {"dram_bytes_per_launch": r["read"] + r["write"], "read": r["read"], "write": r["write"],
              "capture": cap, "kernel": r["kernel"], "duration_us_ncu": r["us"], "round": rnd}
    print(w, doc[w])
json.dump(doc, open(out_p, "w"), indent=1)
