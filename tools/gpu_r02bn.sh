#!/bin/bash
# ncu --set full of the deferred owner-merge pass (late batch of the 1M x 128 build) + source lines
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"owner_merge_kernel<jb::F32Metric, .int.2>" --launch-skip 30 -c 1 \
   -o gpurun_out/prof_owner2_1M -f python tools/exp_build_prof.py > gpurun_out/ncu_owner2.log 2>&1
tail -3 gpurun_out/ncu_owner2.log
python profiles/summarize_ncu.py gpurun_out/prof_owner2_1M.ncu-rep gpurun_out/owner2_summary.txt > /dev/null 2>&1
python profiles/ncu_lines.py gpurun_out/prof_owner2_1M.ncu-rep 45 > gpurun_out/owner2_lines.txt 2>&1
head -60 gpurun_out/owner2_summary.txt
