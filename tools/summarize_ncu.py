#!/usr/bin/env python3
"""Summarise an ncu --set full report into a JSON (per launch: duration,
clocks, DRAM bytes, L2 bytes, tensor-pipe and DRAM utilisation) and, with
--traffic, write profiles/traffic.json (dram read+write per launch keyed
the way bench.py looks it up)."""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "lts__t_bytes.sum", "lts__t_sector_hit_rate.pct",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
        "launch__registers_per_thread", "launch__cluster_dim_x"]
UNIT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:100]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = r[i]
                d[k + ".unit"] = units[i]
        try:
            rd = float(d["dram__bytes_read.sum"]) * UNIT.get(d["dram__bytes_read.sum.unit"], 1)
            wr = float(d["dram__bytes_write.sum"]) * UNIT.get(d["dram__bytes_write.sum.unit"], 1)
            d["dram_bytes_total"] = rd + wr
        except (KeyError, ValueError):
            pass
        res.append(d)
    json.dump(res, open(out, "w"), indent=1)
    if len(sys.argv) > 3 and sys.argv[3] == "--traffic":
        # kernels of the headline bench in launch order: logits (K1), dx (K3), dw (K4)
        names = {"EpiLogitStats": "logits", "<2, 0, 1, vp::EpiStoreF32": "dx", "<2, 1, 1, vp::EpiStoreF32": "dw",
                 "<2, 0, 1, EpiStoreF32": "dx", "<2, 1, 1, EpiStoreF32": "dw"}
        tr = {}
        for d in res:
            for pat, nm in names.items():
                if pat in d["kernel"] and "dram_bytes_total" in d:
                    tr[f"{nm}:8192x4096x256000"] = d["dram_bytes_total"]
        json.dump(tr, open("profiles/traffic.json", "w"), indent=1)
        print("traffic:", tr)
    for d in res:
        print(d["kernel"][:60], d.get("gpu__time_duration.sum"), d.get("gpu__time_duration.sum.unit"),
              "dram", d.get("dram_bytes_total"))


if __name__ == "__main__":
    main()
