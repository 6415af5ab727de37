"""DRAM traffic of one C5 operator pair from an `ncu --set full` capture.

    ncu --set full --clock-control none -k regex:"hot_|seg_adj|head_combine" -s 5 -c 5 \
        -o gpurun_out/c5_pair python scripts/ncu_ops.py 5
    python scripts/ncu_pair_traffic.py gpurun_out/c5_pair.ncu-rep profiles/r2_ncu_c5_pair.json

The capture holds one pair after the warm-up pairs: hot_permute + hot_sell_fwd
(A*v) and the tail / head seg_adj + head_combine (A^T u).  Writes the per-kernel
duration and dram__bytes_read/write and their sum (bench.py's roofline.traffic).
"""
import csv
import io
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}


def val(d, k):
    return float(d[k].replace(",", "")) * scale.get(units[hdr.index(k)], 1.0)


kernels = []
for r in rows[2:]:
    d = dict(zip(hdr, r))
    kernels.append({"kernel": d["Kernel Name"].split("(")[0][-60:],
                    "us": val(d, "gpu__time_duration.sum"),
                    "dram_read": val(d, "dram__bytes_read.sum"),
                    "dram_write": val(d, "dram__bytes_write.sum")})
tot = sum(k["dram_read"] + k["dram_write"] for k in kernels)
json.dump({"source": f"{rep} (ncu --set full, scripts/ncu_ops.py 5: one pair after warm-up)",
           "pair_dram_bytes": tot, "kernels": kernels}, open(out, "w"), indent=1)
print(json.dumps({"pair_dram_bytes": tot, "n_kernels": len(kernels)}))
for k in kernels:
    print(f"{k['us']:9.1f} us  rd {k['dram_read'] / 1e6:9.1f} MB  wr {k['dram_write'] / 1e6:8.1f} MB  {k['kernel']}")
