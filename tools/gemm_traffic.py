"""DRAM traffic of every GEMM launch of one step vs its algorithmic bytes.

    python tools/gemm_traffic.py NCU_CSV SHAPES_CSV OUT_JSON

NCU_CSV: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
-k regex:gemm_tcgen05 --csv` of `tools/profile_step.py --ncu --gemm-shapes SHAPES_CSV`
(launches in issue order == shape rows in order).  Writes the per-launch averages
bench.py reports as roofline.traffic.
"""
import collections, csv, io, json, sys

txt = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(txt) if l.startswith('"ID"'))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3,
         "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}
rows = collections.defaultdict(dict)
for r in csv.DictReader(io.StringIO("\n".join(txt[start:]))):
    rows[int(r["ID"])][r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * scale[r["Metric Unit"]]
launches = [rows[i] for i in sorted(rows)]
shapes = [tuple(int(x) for x in l.split(",")) for l in open(sys.argv[2]) if l.strip()]
if len(shapes) != len(launches):
    sys.exit(f"{len(launches)} ncu launches vs {len(shapes)} logged GEMMs")
per_shape = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
tot_dram = tot_alg = tot_us = 0.0
for (M, N, K, alg), m in zip(shapes, launches):
    dram = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
    e = per_shape[f"{M}x{N}x{K}"]
    e[0] += 1; e[1] += dram; e[2] += alg; e[3] += m["gpu__time_duration.sum"]
    tot_dram += dram; tot_alg += alg; tot_us += m["gpu__time_duration.sum"]
n = len(shapes)
out = {"launches": n, "dram_bytes_per_launch": tot_dram / n, "algorithmic_bytes_per_launch": tot_alg / n,
       "dram_over_algorithmic": tot_dram / tot_alg, "us_per_launch_cold": tot_us / n,
       "shapes": {k: {"launches": c, "dram_bytes_per_launch": d / c, "algorithmic_bytes_per_launch": a / c,
                      "ratio": d / a, "us_per_launch_cold": t / c}
                  for k, (c, d, a, t) in sorted(per_shape.items(), key=lambda kv: -kv[1][3])}}
json.dump(out, open(sys.argv[3], "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k != "shapes"}))
for k, v in out["shapes"].items():
    print(f"{k:>22s} n={v['launches']:4d} dram/alg={v['ratio']:.2f} {v['us_per_launch_cold']:.1f} us")
