#!/bin/bash
# Round-2 GPU session: parity tests, smoke, bench (both arms), the reference's own suite via the stub.
# usage (under gpurun): bash tools/gpu_r02.sh TAG [skip-tests]
TAG=${1:-r02a}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi_$TAG.txt 2>&1
if [ "$2" != "skip-tests" ]; then
  timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
  tail -3 gpurun_out/pytest_gpu_$TAG.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
  tail -2 gpurun_out/smoke_$TAG.log
fi
SECONDS=0; timeout 1500 python bench.py --details gpurun_out/bench_details_$TAG.json > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?"; tail -c 600 gpurun_out/bench_$TAG.json; echo "bench wall $SECONDS s"; tail -5 gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
echo "ref rc=$?"; cat gpurun_out/bench_ref_$TAG.json | head -c 400
echo done
