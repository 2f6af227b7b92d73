#!/usr/bin/env python
"""Write profiles/traffic_config<C>.json from an `ncu --page raw --csv` export of one launch of
the fused degree kernel (bench.py reads it into roofline.traffic).

    python tools/traffic_from_ncu.py gpurun_out/csr_coded_full_raw.csv 3 <algorithmic bytes per launch>
"""
import csv
import json
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    path, cfg, alg = sys.argv[1], int(sys.argv[2]), float(sys.argv[3])
    rows = list(csv.reader(open(path)))
    hdr, units, r = rows[0], rows[1], rows[2]
    idx = {h: i for i, h in enumerate(hdr)}
    get = lambda k: float(r[idx[k]].replace(",", "")) * UNIT[units[idx[k]]]  # noqa: E731
    rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
    out = {"dram_bytes_per_launch": int(rd + wr), "kernel": r[idx["Kernel Name"]],
           "source": f"{path}: ncu --set full --clock-control none, one launch: dram__bytes_read.sum "
                     f"{rd / 1e6:.1f} MB + dram__bytes_write.sum {wr / 1e6:.1f} MB",
           "algorithmic_bytes_per_launch": int(alg), "traffic_over_algorithmic": round((rd + wr) / alg, 4)}
    json.dump(out, open(f"profiles/traffic_config{cfg}.json", "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
