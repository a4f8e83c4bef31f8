"""Refresh profiles/ncu_summary.json["k_jacobi_c2"] (the entry bench.py reads for
roofline.traffic) from an `ncu --page raw --csv` export of the finest k_jacobi capture
(tools/profile_round.sh writes gpurun_out/prof/k_jacobi_c2_raw.csv).

    python tools/ncu_summary_update.py gpurun_out/prof/k_jacobi_c2_raw.csv "<build / round note>"
"""
import csv
import json
import sys

raw, note = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(raw)))
d = dict(zip(rows[0], rows[2]))


def f(key):
    return float(d[key].replace(",", ""))


def to_bytes(key):  # the raw page prints dram bytes in the unit row's unit
    unit = dict(zip(rows[0], rows[1]))[key].lower()
    scale = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}[unit]
    return int(round(f(key) * scale))


path = "profiles/ncu_summary.json"
s = json.load(open(path))
old = s["k_jacobi_c2"]
rd, wr = to_bytes("dram__bytes_read.sum"), to_bytes("dram__bytes_write.sum")
dur_unit = dict(zip(rows[0], rows[1]))["gpu__time_duration.sum"].lower()
dur = f("gpu__time_duration.sum") * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}[dur_unit]
s["k_jacobi_c2"] = {
    "source": f"profiles/r02_ncu_k_jacobi_c2_raw.csv ({note}: ncu --set full --clock-control none, "
              "tools/profile_round.sh, 4th finest-level k_jacobi launch of tools/profile_sweep.py 7 0)",
    "duration_us_ncu": round(dur, 3),
    "dram_bytes_read": rd,
    "dram_bytes_write": wr,
    "dram_bytes_per_launch": rd + wr,
    "stored_bytes_per_launch": old["stored_bytes_per_launch"],
    "registers_per_thread": int(f("launch__registers_per_thread")),
    "achieved_occupancy_pct": round(f("sm__warps_active.avg.pct_of_peak_sustained_active"), 2),
    "l1tex_throughput_pct": round(f("l1tex__throughput.avg.pct_of_peak_sustained_elapsed"), 2),
    "l2_hit_rate_pct": round(f("lts__t_sector_hit_rate.pct"), 2),
    "dram_throughput_pct_of_ncu_peak": round(f("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"), 2),
    "warp_cycles_per_issued_instruction": round(f("smsp__average_warp_latency_per_inst_issued.ratio"), 2),
}
json.dump(s, open(path, "w"), indent=1)
print(json.dumps(s["k_jacobi_c2"], indent=1))
