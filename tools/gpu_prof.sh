#!/bin/bash
# ncu --set full of chosen network layers (exact bench arguments): bash tools/gpu_prof.sh TAG NET BATCH SCHEME LAYERS
# reports stay on the box (/tmp); text summaries come back under gpurun_out/
TAG=$1; NET=$2; B=$3; SCH=$4; LAYERS=$5
mkdir -p gpurun_out
ABFT_TRACE=1 timeout 600 python tools/ncu_netlayer.py $NET $B $SCH $LAYERS 1 > gpurun_out/times_$TAG.log 2>&1
grep -v "^\[abft\]" gpurun_out/times_$TAG.log | head -20
N=$(echo $LAYERS | tr ',' '\n' | wc -l)
ABFT_TRACE=1 timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -c $((N*2)) \
  -o /tmp/full_$TAG -f python tools/ncu_netlayer.py $NET $B $SCH $LAYERS 1 > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_$TAG.log
python tools/ncu_summary.py /tmp/full_$TAG.ncu-rep l2 lts__t_bytes.sum smsp__pcsamp > gpurun_out/ncu_sum_$TAG.txt 2>&1
ncu -i /tmp/full_$TAG.ncu-rep --page details --csv > gpurun_out/ncu_details_$TAG.csv 2>/dev/null
python tools/ncu_stalls.py /tmp/full_$TAG.ncu-rep > gpurun_out/ncu_stalls_$TAG.txt 2>&1
python tools/ncu_pipes.py /tmp/full_$TAG.ncu-rep > gpurun_out/ncu_pipes_$TAG.txt 2>&1
