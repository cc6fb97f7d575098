"""Summarise ncu --set full reports into profiles/<round>/traffic.json:
DRAM bytes read / written, duration, DRAM and SM throughput per kernel, keyed
by config then by the bench's kernel names (dense_decode / fast_decode).

    python scripts/ncu_traffic.py profiles/r02/traffic.json c2=gpurun_out/x.ncu-rep c4=...
"""
import csv
import io
import json
import subprocess
import sys

NAMES = {"decode_tc_kernel": "dense_decode", "decode_kernel": "dense_decode", "fast_decode_kernel": "fast_decode"}
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__registers_per_thread"]
UNIT = {"dram__bytes_read.sum": None, "dram__bytes_write.sum": None}


def scale(v, unit):
    f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(unit, 1)
    return float(v.replace(",", "")) * f


def main():
    out_path = sys.argv[1]
    try:
        with open(out_path) as f:
            res = json.load(f)
    except FileNotFoundError:
        res = {}
    for arg in sys.argv[2:]:
        cfg, rep = arg.split("=", 1)
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            name = r[hdr.index("Kernel Name")]
            key = next((v for k, v in NAMES.items() if f"::{k}<" in name or f"::{k}(" in name), None)
            if key is None:
                continue
            e = {"kernel": name[:120]}
            for m in METRICS:
                if m in hdr:
                    i = hdr.index(m)
                    e[m] = scale(r[i], units[i])
            e["dram_read_bytes"] = e.get("dram__bytes_read.sum")
            e["dram_write_bytes"] = e.get("dram__bytes_write.sum")
            e["duration_us"] = e.get("gpu__time_duration.sum")
            res.setdefault(cfg, {})[key] = e  # last launch of each kind
    with open(out_path, "w") as f:
        json.dump(res, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
