timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/t_14.log 2>&1; tail -3 gpurun_out/t_14.log
SECONDS=0; timeout 1500 python bench.py --details gpurun_out/bench_details_r02e.json > gpurun_out/bench_r02e.json 2> gpurun_out/bench_r02e.err
echo "bench rc=$? wall $SECONDS s"; tail -c 700 gpurun_out/bench_r02e.json; tail -3 gpurun_out/bench_r02e.err
