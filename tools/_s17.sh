SECONDS=0; timeout 1500 python bench.py --details gpurun_out/bench_details_r02f.json > gpurun_out/bench_r02f.json 2> gpurun_out/bench_r02f.err
echo "bench rc=$? wall $SECONDS s"; tail -c 900 gpurun_out/bench_r02f.json; tail -3 gpurun_out/bench_r02f.err
