"""Summarise an `ncu --page raw --csv` + `--page source --csv` pair: key counters, stall
reasons per issued instruction, and the SASS lines with the most stall samples.
Usage: python tools/ncu_stalls.py <raw.csv> <source.csv> [top]"""
import csv
import sys


def main():
    raw, src = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    rows = list(csv.reader(open(raw)))
    hdr, r = rows[0], rows[2]
    col = {h: i for i, h in enumerate(hdr)}
    for k in ["Kernel Name", "gpu__time_duration.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
              "sm__cycles_active.avg", "sm__cycles_elapsed.avg", "smsp__warps_eligible.avg.per_cycle_active",
              "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__warps_active.avg.per_cycle_active",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum"]:
        if k in col:
            print(f"{k}: {r[col[k]]}")
    for h, i in col.items():
        if "issue_stalled" in h and h.endswith("per_issue_active.ratio") and float(r[i] or 0) > 0.05:
            print(f"  stall {h.split('issue_stalled_')[1].split('_per_issue')[0]}: {float(r[i]):.2f}")
    rows = list(csv.reader(open(src)))
    while rows and (not rows[0] or rows[0][0] != "Address"):
        rows.pop(0)
    hdr = rows[0]
    col = {h: i for i, h in enumerate(hdr)}
    samp = "Warp Stall Sampling (All Samples)"
    data = []
    for row in rows[1:]:
        try:
            data.append((int(row[col[samp]] or 0), row))
        except ValueError:
            pass
    total = sum(d[0] for d in data)
    print(f"total samples {total} ({samp})")
    stall_cols = [h for h in hdr if h.startswith("stall_")]
    for n, row in sorted(data, key=lambda d: -d[0])[:top]:
        reasons = sorted(((int(row[col[h]] or 0), h) for h in stall_cols), reverse=True)[:3]
        print(f"{100.0 * n / total:5.1f}%  {row[col['Source']][:70]:70s}  " +
              ", ".join(f"{h[6:]}={v}" for v, h in reasons if v))


if __name__ == "__main__":
    main()
