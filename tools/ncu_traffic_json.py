"""Per-launch DRAM traffic of one lockstep step from an ncu --set full capture
(light + step + overflow kernels of one step) -> profiles/ncu_step_kernel*.json,
the `roofline.traffic` source bench.py reads.  Run here (no GPU needed).

usage: python tools/ncu_traffic_json.py REPORT.ncu-rep OUT.json "source description"
"""
import csv
import json
import subprocess
import sys


def main(path, out, source):
    txt = subprocess.check_output(["ncu", "-i", path, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    col = {n: i for i, n in enumerate(hdr)}
    kernels = {}

    def val(row, name):
        v = float(row[col[name]].replace(",", ""))
        u = units[col[name]]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3,
                 "usecond": 1, "msecond": 1e3, "ns": 1e-3, "us": 1, "ms": 1e3, "inst": 1, "": 1}
        if u not in scale:
            raise ValueError(f"unknown unit {u!r} for {name}")
        scale = scale[u]
        return v * scale

    for row in rows[2:]:
        name = row[col["Kernel Name"]].split("(")[0].split("::")[-1]
        kernels[name] = {"dram_bytes_read": val(row, "dram__bytes_read.sum"),
                         "dram_bytes_write": val(row, "dram__bytes_write.sum"),
                         "duration_us_cold": val(row, "gpu__time_duration.sum"),
                         "warp_instructions": val(row, "smsp__inst_executed.sum")}
    total = sum(k["dram_bytes_read"] + k["dram_bytes_write"] for k in kernels.values())
    inst = sum(k["warp_instructions"] for k in kernels.values())
    json.dump({"source": source, "kernels": kernels, "warp_instructions_per_launch": inst,
               "kernel": "one lockstep step = rkc_light_kernel + rkc_step_kernel + rkc_step_overflow_kernel",
               "dram_bytes_per_launch": total}, open(out, "w"), indent=1)
    print(json.dumps(kernels, indent=1), total)


if __name__ == "__main__":
    main(*sys.argv[1:4])
