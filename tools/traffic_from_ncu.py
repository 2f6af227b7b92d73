#!/usr/bin/env python
"""Write profiles/traffic_config<C>.json from an `ncu --page raw --csv` export of one launch of
the fused degree kernel (bench.py reads it into roofline.traffic).

    python tools/traffic_from_ncu.py <raw.csv> <config> <algorithmic bytes per launch> <matrix bytes> <k>

<matrix bytes> = npc_operator_matrix_bytes of the operator profiled: bench.py uses the figure
only while the operator it builds stores the same number of bytes (same format).
"""
import csv
import json
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    path, cfg, alg = sys.argv[1], int(sys.argv[2]), float(sys.argv[3])
    mbytes = float(sys.argv[4]) if len(sys.argv) > 4 else None
    k = int(sys.argv[5]) if len(sys.argv) > 5 else None
    rows = list(csv.reader(open(path)))
    hdr, units, r = rows[0], rows[1], rows[2]
    idx = {h: i for i, h in enumerate(hdr)}
    get = lambda k: float(r[idx[k]].replace(",", "")) * UNIT[units[idx[k]]]  # noqa: E731
    rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
    out = {"dram_bytes_per_launch": int(rd + wr), "kernel": r[idx["Kernel Name"]],
           "source": f"{path}: ncu --set full --clock-control none, one launch: dram__bytes_read.sum "
                     f"{rd / 1e6:.1f} MB + dram__bytes_write.sum {wr / 1e6:.1f} MB",
           "algorithmic_bytes_per_launch": int(alg), "traffic_over_algorithmic": round((rd + wr) / alg, 4),
           "matrix_bytes": mbytes, "k": k}
    for key in ("lts__t_sectors.sum", "lts__t_sectors_srcunit_tex.sum", "lts__t_sectors_srcunit_ltcfabric.sum",
                "gpu__time_duration.sum"):
        if key in idx:
            out[key] = float(r[idx[key]].replace(",", ""))
    json.dump(out, open(f"profiles/traffic_config{cfg}.json", "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
