#!/bin/bash
# Round-2 evidence on one GPU box (all text summaries land in gpurun_out/, copied to profiles/ by hand):
#   bench line (both arms), the ncu launch list of one timed IG step, and --set full summaries of
#   the dominant kernels (one report per layer: VGG-16 conv1_2 = the step's longest launch, a
#   compute-bound VGG-16 conv, the FC 25088->4096, the gathered ResNet-50 stem, a residual conv).
TAG=${1:-r02}
mkdir -p gpurun_out
SECONDS=0
timeout 1500 python bench.py --details gpurun_out/bench_details_$TAG.json > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$? wall $SECONDS s"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference_$TAG.json 2>&1
timeout 1500 ncu --nvtx --nvtx-include "timed_ig/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 3 --no-secondary > gpurun_out/bench_ncu_$TAG.log 2>&1
echo "launch list rc=$?"
prof() {   # NAME NET LAYER SCHEME [dominant]
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -c 1 \
    -o /tmp/p_$1 -f python tools/ncu_netlayer.py $2 256 $4 $3 1 > gpurun_out/ncu_log_$1.log 2>&1
  if [ -n "$5" ]; then
    python tools/ncu_layer_summary.py /tmp/p_$1.ncu-rep "$2 b256 $3 $4" $2 $3 256 $4 > gpurun_out/ncu_$1.txt 2>&1
  else
    python tools/ncu_layer_summary.py /tmp/p_$1.ncu-rep "$2 b256 $3 $4" > gpurun_out/ncu_$1.txt 2>&1
  fi
  python tools/ncu_stalls.py /tmp/p_$1.ncu-rep > gpurun_out/ncu_stalls_$1.txt 2>&1
  echo "prof $1 done"
}
prof vgg_conv1_2 vgg16 features.2 global-abft dominant
prof vgg_conv3_2 vgg16 features.14 global-fused
prof vgg_conv3_2_unprot vgg16 features.14 unprotected
prof vgg_fc6 vgg16 classifier.0 global-abft
prof rn_stem resnet50 conv1 global-abft
prof rn_l1_conv3 resnet50 layer1.0.conv3 unprotected
echo done
