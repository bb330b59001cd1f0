"""Write profiles/ncu_traffic.json from an `ncu --page raw --csv` export of one
launch of the bench step's fused kernel (ws2_kernel since round 2): DRAM
bytes and warp instructions per launch, read by bench.py's roofline.

    ncu -i gpurun_out/ev_ws.ncu-rep --page raw --csv > raw.csv
    python tools/update_traffic.py raw.csv "<source note>"
"""
import csv
import json
import os
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "inst": 1, "": 1}


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    h, units, vals = rows[0], rows[1], rows[2]

    def get(name):
        i = h.index(name)
        return float(vals[i].replace(",", "")) * UNITS.get(units[i], 1)

    rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
    inst = get("smsp__inst_executed.sum")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = os.path.join(root, "profiles", "ncu_traffic.json")
    d = {"C3": {"scan_kernel_dram_bytes_per_launch": int(round(rd + wr)),
                "smsp_inst_executed_per_launch": int(round(inst)),
                "dram_read_bytes": int(round(rd)), "dram_write_bytes": int(round(wr)),
                "algorithmic_bytes_per_launch": 768000000,
                "source": sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]}}
    json.dump(d, open(out, "w"), indent=1)
    print(json.dumps(d))


if __name__ == "__main__":
    main()
