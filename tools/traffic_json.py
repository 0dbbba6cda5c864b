"""Roofline inputs for bench.py from one `ncu --set full` capture of ONE focus_score call
(every k_* launch of it): DRAM bytes per image of the dominant kernel and of the whole
step, and the dominant kernel's tensor-pipe activity.
Usage: python tools/traffic_json.py report.ncu-rep <images per call> <kernel> <source text>
       > profiles/ncu_<kernel>_traffic.json"""
import csv
import io
import json
import subprocess
import sys

rep, images, kernel, source = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def num(d, u, k):
    return float(d[k].replace(",", "")) * scale.get(u[k], 1.0)


per_kernel, step = {}, 0.0
res = {"kernel": kernel, "source": source, "images": images}
for vals in rows[2:]:
    d, u = dict(zip(hdr, vals)), dict(zip(hdr, units))
    name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("mhfd::", "")
    if not name.startswith("k_"):
        continue
    b = num(d, u, "dram__bytes_read.sum") + num(d, u, "dram__bytes_write.sum")
    per_kernel[name] = per_kernel.get(name, 0.0) + b
    step += b
    if name.startswith(kernel + "<") or name == kernel:
        res["dram_bytes_read"] = num(d, u, "dram__bytes_read.sum")
        res["dram_bytes_write"] = num(d, u, "dram__bytes_write.sum")
        res["dram_bytes_per_image"] = (res["dram_bytes_read"] + res["dram_bytes_write"]) / images
        k = "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
        if k in d:
            res["tensor_active_pct"] = float(d[k])
        tsc = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
        res["duration_ms"] = float(d["gpu__time_duration.sum"].replace(",", "")) * tsc[u["gpu__time_duration.sum"]]
res["step_dram_bytes_per_image"] = step / images
res["per_kernel_dram_bytes_per_image"] = {k: v / images for k, v in per_kernel.items()}
print(json.dumps(res, indent=1))
