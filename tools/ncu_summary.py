"""Builds profiles/rNN_ncu_summary.json (the bench line's roofline.traffic) from a
committed raw ncu export (`ncu -i X.ncu-rep --page raw --csv > profiles/rNN_..._raw.csv`),
so the traffic figure is reproducible from the capture it comes from.

    python tools/ncu_summary.py profiles/r02_ncu_group_tma_pack_raw.csv profiles/r02_ncu_summary.json
"""
import csv
import json
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main(src, dst):
    rows = list(csv.reader(open(src)))
    h, units = rows[0], rows[1]
    k, rd, wr, t = (h.index(c) for c in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                          "gpu__time_duration.sum"))
    mul_sum = []
    out = {"source": f"{src}: ncu --set full --clock-control none -k regex:\"group_tma|tma_pack\" "
                     "(bench.py --steps 1 --warmup 1 --skip-e2e --skip-cpu --skip-extra)",
           "launches": []}
    for r in rows[2:]:
        b = float(r[rd]) * UNIT[units[rd]] + float(r[wr]) * UNIT[units[wr]]
        name = r[k].split("(")[0]
        out["launches"].append({"kernel": name, "dram_bytes": b, "ms": float(r[t])})
        if "group_tma" in name:
            mul_sum.append(b)
        if "tma_pack" in name:
            out["c5_pack_bytes_per_launch"] = b
    out["c5_mul_sum_bytes_per_launch"] = sum(mul_sum) / len(mul_sum)
    # one step = the three fused products (dims 1, 2, 3); the capture may hold several steps
    out["c5_mul_sum_bytes_per_step"] = sum(mul_sum) / (len(mul_sum) / 3)
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
