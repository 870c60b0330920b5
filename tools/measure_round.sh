#!/bin/bash
# One GPU pass of the round's measurements (run under gpurun from the repo root):
# the bench line, the reference arm, the bench's kernel launch list, the raw
# ncu export behind roofline.traffic, and a full capture of the config-3 chain.
# Outputs land in gpurun_out/ (the ncu reports in /tmp: gpurun copies back <= 64 MiB);
# the judged copies go to profiles/ by hand.
set -u
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo "ref rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --skip-e2e --skip-cpu \
    --skip-extra > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
ncu --set full --clock-control none -k regex:"group_tma|tma_pack" -o /tmp/c5_full -f \
    python bench.py --steps 1 --warmup 1 --skip-e2e --skip-cpu --skip-extra > gpurun_out/ncu_c5.log 2>&1
ncu -i /tmp/c5_full.ncu-rep --page raw --csv > gpurun_out/c5_raw.csv 2>&1
echo "c5 full rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"fold_gemm_ws|col_tree|row_tree" -s 8 -c 4 \
    -o /tmp/c3b_full -f python tools/one_c3b_chain.py > gpurun_out/ncu_c3b.log 2>&1
ncu -i /tmp/c3b_full.ncu-rep --page raw --csv > gpurun_out/c3b_raw.csv 2>&1
echo "c3b full rc=$?"
