#!/bin/bash
# ncu source-level capture of one slot_gemm micro configuration: tools/ncu_sg.sh <config index> <tag>
idx=$1; tag=$2
SG_ONLY=$idx ncu --set full --import-source on --clock-control none --kernel-name regex:sg_kernel --launch-skip 2 --launch-count 1 -f -o /tmp/sg_$tag ./tools/micro/slot_gemm > gpurun_out/ncu_sg_$tag.log 2>&1
ncu -i /tmp/sg_$tag.ncu-rep --page source --csv > gpurun_out/sg_${tag}_source.csv 2>/dev/null
ncu -i /tmp/sg_$tag.ncu-rep --page raw --csv > gpurun_out/sg_${tag}_raw.csv 2>/dev/null
