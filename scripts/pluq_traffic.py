"""DRAM traffic of the tensor-core GEMM launches inside one PLUQ, from an ncu metrics capture.

    FFG_GEMM_LOG=1 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --clock-control none -k regex:modgemm --csv --log-file gemm_dram.csv \
        python scripts/gemm_shapes.py --run --n 16384 2> shapes.log
    python scripts/pluq_traffic.py gemm_dram.csv shapes.log --n 16384 --p 131071 --thr 64 \
        > profiles/pluq_gemm_traffic.json

Algorithmic bytes per launch: A and B read once (4 bytes per residue for the direct kernel,
K <= 256; L limb bytes for the TMA kernel) plus C read and written once (4 + 4 bytes per residue)
-- the GEMM kernel's own operands, not the split pass.
"""
import argparse
import csv
import json

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("shapes")
ap.add_argument("--n", type=int, required=True)
ap.add_argument("--p", type=int, required=True)
ap.add_argument("--thr", type=int, required=True)
a = ap.parse_args()

limbs = max(1, ((a.p - 1).bit_length() + 7) // 8)
rows = [r for r in csv.reader(l for l in open(a.csv) if l.startswith('"'))]
hdr, body = rows[0], rows[1:]
ci = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value")}
per = {}
for r in body:
    if "modgemm" not in r[ci["Kernel Name"]] or "simt" in r[ci["Kernel Name"]]:
        continue
    v = float(r[ci["Metric Value"]].replace(",", ""))
    name = r[ci["Metric Name"]]
    unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else ""
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(unit, 1)
    per.setdefault(r[ci["ID"]], {})[name] = v * scale
launches = len(per)
dram = sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in per.values())
ns = sum(d.get("gpu__time_duration.sum", 0) for d in per.values())

algo = 0.0
tc = 0
on = False
for line in open(a.shapes):
    if line.startswith("FFG_GEMM_BEGIN"):
        on, algo, tc = True, 0.0, 0
    elif on and line.startswith("FFG_GEMM "):
        m, nn, k, simt = map(int, line.split()[1:])
        if simt:
            continue
        tc += 1
        # direct kernel (K <= 256) reads the u32 operands; the TMA kernel reads limb planes
        opb = 4 if k <= 256 else limbs
        algo += opb * (m * k + k * nn) + 8.0 * m * nn
out = {"n": a.n, "p": a.p, "threshold": a.thr, "limbs": limbs, "modgemm_launches": launches,
       "tc_gemm_calls_logged": tc,
       "dram_bytes_per_launch": dram / launches if launches else None,
       "algorithmic_bytes_per_launch": algo / tc if tc else None,
       "dram_over_algorithmic": (dram / launches) / (algo / tc) if launches and tc and algo else None,
       "ncu_serialized_gemm_ms": ns / 1e6,
       "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                 "-k regex:modgemm over one PLUQ (scripts/pluq_traffic.py)"}
print(json.dumps(out, indent=1))
