#!/bin/bash
# Round-2 evidence on one GPU box (all text summaries land in gpurun_out/, copied to profiles/ by hand):
#   bench line (both arms), the ncu launch list of one timed IG step, and --set full summaries of
#   the dominant kernel (the IG plan's longest launch, with the plan the bench chose: variant and
#   plan flags from the bench line) plus a compute-bound VGG-16 conv, the FC 25088->4096, the
#   gathered ResNet-50 stem and a residual conv.
TAG=${1:-r02}
mkdir -p gpurun_out
SECONDS=0
timeout 1500 python bench.py --details gpurun_out/bench_details_$TAG.json > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$? wall $SECONDS s"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference_$TAG.json 2>&1
timeout 1500 ncu --nvtx --nvtx-include "timed_ig/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 3 --no-secondary > gpurun_out/bench_ncu_$TAG.log 2>&1
echo "launch list rc=$?"
prof() {   # NAME NET LAYER SCHEME FLAGS [dominant: bench-scheme variant]
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -c 1 \
    -o /tmp/p_$1 -f python tools/ncu_netlayer.py $2 256 $4 $3 1 $5 > gpurun_out/ncu_log_$1.log 2>&1
  if [ -n "$6" ]; then
    python tools/ncu_layer_summary.py /tmp/p_$1.ncu-rep "$2 b256 $3 $4 flags $5" $2 $3 256 $6 $5 $7 > gpurun_out/ncu_$1.txt 2>&1
  else
    python tools/ncu_layer_summary.py /tmp/p_$1.ncu-rep "$2 b256 $3 $4 flags $5" > gpurun_out/ncu_$1.txt 2>&1
  fi
  python tools/ncu_stalls.py /tmp/p_$1.ncu-rep > gpurun_out/ncu_stalls_$1.txt 2>&1
  echo "prof $1 done"
}
read NET LAYER SCHEME LSCHEME VAR FLAGS < <(python - "gpurun_out/bench_$TAG.json" <<'PY'
import json, re, sys
k = json.load(open(sys.argv[1]))["roofline"]["kernel"]
net, layer, scheme, var, tile, flags = re.match(
    r"abft_gemm_kernel (\S+) (\S+) (\S+) .*variant=(\S+) tile_n=(\d+) flags=(\d+)", k).groups()
lsch = {"dot": "global-dot", "fused": "global-fused"}.get(var, scheme) if scheme == "global-abft" else scheme
print(net, layer, scheme, lsch, var, flags)
PY
)
echo "dominant: $NET $LAYER $SCHEME ($LSCHEME) flags $FLAGS"
prof dominant $NET $LAYER $LSCHEME $FLAGS $SCHEME $VAR
prof vgg_conv4_2_pair vgg16 features.19 global-fused 6144
prof vgg_conv4_2_pair_unprot vgg16 features.19 unprotected 6144
prof vgg_fc6 vgg16 classifier.0 global-abft 0
prof rn_stem resnet50 conv1 global-abft 0
prof rn_l1_conv3 resnet50 layer1.0.conv3 unprotected 0
echo done
