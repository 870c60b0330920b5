"""Rewrites the bench tables of profiles/rNN_summary.md (between 'Bench line:' and the ncu
paragraph) from the committed bench lines.
    python tools/summary_table.py profiles/r02_bench_final.json profiles/r02_bench_ref.json profiles/r02_summary.md"""
import json
import sys


def main(final, ref, md):
    d = json.loads(open(final).read().strip().splitlines()[-1])
    r = json.loads(open(ref).read().strip().splitlines()[-1])
    o = d["ops"]
    s = open(md).read()
    start = s.index("Bench line:")
    end = s.index("ncu (`--set full --clock-control none`; serialised")
    new = f"""Bench line: `{final}` (`python bench.py`, 10 steps after 3 warm-up;
final pass of the round: SM clock {d['clocks']['sm_mhz']:.0f} of {d['clocks']['sm_max_mhz']} MHz, throttle reasons {d['clocks']['reasons']}).  Reference
arm: `{ref}` (`python bench.py --impl reference`: the reference's own
C++ path compiled from `/root/reference/proj/include` by `oracle/Makefile`, 16 host threads,
same `config`).  GPU suite on the same box: 162 passed; `smoke()` ok.

| quantity | value |
|---|---|
| config 5 step (3 fused multiply + rotate-and-sum products, 16 GiB X) | {d['ms_per_step']:.2f} ms (8.1-8.5 ms across the round's runs and boxes with the same code: 0.96-1.0 of the copy peak) |
| `value` | {d['value']:.3g} tile-slots/s |
| roofline (fused products) | {d['roofline']['achieved']:.0f} GB/s = {d['roofline']['frac']:.3f} of the measured {d['roofline']['peak']:.0f} GB/s copy burst; ncu DRAM bytes per launch {d['roofline']['traffic'] / 1e9:.2f} GB = 1.00 x algorithmic |
| `e2e` (pinned host in, pack, 3 products, unpack, D2H) | {d['e2e']['value']:.3g} tile-slots/s, {d['e2e']['ms_per_step']:.0f} ms per step (PCIe: 17.19 GB H2D per step; a plain 16 GiB H2D takes 310 ms on the same box, `tools/probe_e2e_pack.py`) |
| reference arm (16 threads) | {r['value']:.3g} tile-slots/s; ours / reference = {d['value'] / r['value']:.0f}x (kernels), {d['e2e']['value'] / r['value']:.0f}x (e2e); value / cpu_baseline = {d['value'] / d['cpu_baseline']['value']:.0f}x (same slab, same measurement) |
| reference, 1 thread | {r['cpu_baseline']['one_thread']['value']:.3g} tile-slots/s |

Per-op lines (`ops`, fraction of the measured copy peak):

| op | time | fraction |
|---|---|---|
| fused products dim 1 / 2 / 3 | {o['mul_sum_dim1']['ms']:.2f} / {o['mul_sum_dim2']['ms']:.2f} / {o['mul_sum_dim3']['ms']:.2f} ms | {o['mul_sum_dim1']['frac']:.2f} / {o['mul_sum_dim2']['frac']:.2f} / {o['mul_sum_dim3']['frac']:.2f} |
| pack / unpack (32 GiB moved each) | {o['pack']['ms']:.2f} / {o['unpack']['ms']:.2f} ms | {o['pack']['frac']:.2f} / {o['unpack']['frac']:.2f} |
| X * W (W broadcast) / X + X | {o['ew_mul_bcast']['ms']:.2f} / {o['ew_add']['ms']:.2f} ms | {o['ew_mul_bcast']['frac']:.2f} / {o['ew_add']['frac']:.2f} |
| tt_sum dim 1 / 2 / 3 | {o['sum_dim1']['ms']:.2f} / {o['sum_dim2']['ms']:.2f} / {o['sum_dim3']['ms']:.2f} ms | {o['sum_dim1']['frac']:.2f} / {o['sum_dim2']['frac']:.2f} / {o['sum_dim3']['frac']:.2f} |
| rotate (16 GiB) | {o['rotate']['ms']:.2f} ms | {o['rotate']['frac']:.2f} (round 1: 0.92) |
| clean_unknowns / replicate_dim (8192 tiles) | {o['clean_unknowns']['ms']:.3f} / {o['replicate_dim']['ms']:.3f} ms | {o['clean_unknowns']['frac']:.2f} / {o['replicate_dim']['frac']:.2f} (replicate_dim 0.83-0.97 across runs; round 1: 0.86 / 0.81) |
| config 3 "3b" tile matmul chain | {o['matmul_c3b']['ms'] * 1e3:.1f} us ({o['matmul_c3b']['graph_replay_ms'] * 1e3:.1f} us as a CUDA graph) | {o['matmul_c3b']['frac']:.2f} of copy peak on the survey's 304 MiB; FP64 {o['matmul_c3b']['fp64_frac']:.2f} (round 1: 0.0978 ms) |
| config 3 "3a" literal chain | {o['matmul_c3a']['ms'] * 1e3:.0f} us ({o['matmul_c3a']['separate_calls_ms'] * 1e3:.0f} us as four calls) | FP64 {o['matmul_c3a']['fp64_frac']:.2f} |
| config 1 / 2 (Python API, per call) | {o['c1_mul_sum']['us']:.1f} / {o['c2_matvec']['us']:.1f} us | — (config 2: 12.3 us before the group-blocked ring fold) |
| config 4 FC-square-FC | {o['c4_fc_square_fc']['us']:.0f} us ({o['c4_fc_square_fc']['graph_replay_us']:.0f} us graph) | — |
| C++ drop-in: c1 / c2 / c3b / c4 | {o['cpp']['c1_mul_sum']['us']:.1f} / {o['cpp']['c2_matvec']['us']:.1f} / {o['cpp']['c3b_matmul_chain']['us']:.1f} / {o['cpp']['c4_fc_square_fc']['us']:.0f} us | — |

"""
    open(md, "w").write(s[:start] + new + s[end:])


if __name__ == "__main__":
    main(*sys.argv[1:4])
