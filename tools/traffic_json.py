"""profiles/rNN/traffic.json: DRAM bytes (read + write) per launch of each config's dominant
kernel, from the round's ncu --set full exports (ncu_full_<name>_raw.csv) and, for launch chains
(config 3's per-class grids), the whole-chain range measurement (range_cfgN.csv).
    python tools/traffic_json.py profiles/r02"""
import csv
import io
import json
import os
import sys

WORKLOADS = {"cfg1_stage": "cfg1_n16_c1_r2", "cfg2_stage": "cfg2_n16_c35_r3", "cfg4_klt": "cfg4_klt_n64_c35",
             "cfg5_gemm": "cfg5_n256_c35_r4", "cfg3_clsjit": "cfg3_n64_c35_r4"}


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def kernels(path):
    rows = list(csv.reader(open(path)))
    h, units = rows[0], rows[1]
    for d in rows[2:]:
        rec = dict(zip(h, d))
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            rec[k] = float(rec[k].replace(",", "")) * SCALE.get(units[h.index(k)], 1)
        yield rec, units


def main(dirname):
    out = {}
    for name, wl in WORKLOADS.items():
        p = os.path.join(dirname, f"ncu_full_{name}_raw.csv")
        if not os.path.exists(p):
            continue
        rs = [d for d, _ in kernels(p)]
        rd = sum(d["dram__bytes_read.sum"] for d in rs) / len(rs)
        wr = sum(d["dram__bytes_write.sum"] for d in rs) / len(rs)
        out[wl] = {"kernel": rs[0]["Kernel Name"][:120], "launches_averaged": len(rs),
                   "dram_bytes_read": rd, "dram_bytes_write": wr, "traffic_bytes_per_launch": rd + wr,
                   "source": f"{os.path.relpath(p)} (ncu --set full --clock-control none)"}
    for c, wl in [(2, "cfg2_n16_c35_r3"), (3, "cfg3_n64_c35_r4"), (4, "cfg4_klt_n64_c35"), (5, "cfg5_n256_c35_r4")]:
        p = os.path.join(dirname, f"range_cfg{c}.csv")
        if not os.path.exists(p) or os.path.getsize(p) == 0:
            continue
        txt = open(p).read()
        txt = txt[txt.index('"ID"'):] if '"ID"' in txt else txt
        vals = {}
        for d in csv.DictReader(io.StringIO(txt)):
            try:
                v = float(d["Metric Value"].replace(",", ""))
            except (KeyError, ValueError):
                continue
            unit = d.get("Metric Unit", "")
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(unit, 1)
            vals[d["Metric Name"]] = vals.get(d["Metric Name"], 0.0) + v * scale
        if "dram__bytes_read.sum" in vals:
            entry = {"range_dram_bytes_read": vals["dram__bytes_read.sum"],
                     "range_dram_bytes_write": vals.get("dram__bytes_write.sum", 0.0),
                     "range_source": f"{os.path.relpath(p)} (ncu --replay-mode range over one forward call)"}
            out.setdefault(wl, {}).update(entry)
            if wl == "cfg3_n64_c35_r4" or "traffic_bytes_per_launch" not in out[wl]:
                out[wl]["traffic_bytes_per_launch"] = entry["range_dram_bytes_read"] + entry["range_dram_bytes_write"]
                out[wl]["source"] = entry["range_source"]
    with open(os.path.join(dirname, "traffic.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1)[:1500])


if __name__ == "__main__":
    main(sys.argv[1])
