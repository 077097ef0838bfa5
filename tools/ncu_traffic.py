"""Fold `ncu --page raw --csv` exports into profiles/ncu_traffic.json:
{config: {stage: dram_read+dram_write bytes per launch}} (bench.py's
roofline.traffic).  Usage: python tools/ncu_traffic.py c2=path_raw.csv ..."""
import csv
import json
import sys
from pathlib import Path

OUT = Path(__file__).resolve().parent.parent / "profiles" / "ncu_traffic.json"
STAGE = {"k_input": "input_xform", "k_gemm": "gemm", "k_output": "output_xform"}


def scale(v, unit):
    return float(v.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]


def main(args):
    data = json.loads(OUT.read_text()) if OUT.exists() else {}
    for a in args:
        cfg, path = a.split("=", 1)
        rows = list(csv.reader(open(path)))
        h, units = rows[0], rows[1]
        ri, wi, ki = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum"), h.index("Kernel Name")
        for r in rows[2:]:
            for key, stage in STAGE.items():
                if key in r[ki]:
                    data.setdefault(cfg, {})[stage] = round(scale(r[ri], units[ri]) + scale(r[wi], units[wi]))
    OUT.write_text(json.dumps(data, indent=1, sort_keys=True) + "\n")
    print(json.dumps(data, indent=1))


if __name__ == "__main__":
    main(sys.argv[1:])
