SECONDS=0; timeout 1500 python bench.py --details gpurun_out/bench_details_r02d.json > gpurun_out/bench_r02d.json 2> gpurun_out/bench_r02d.err
echo "bench rc=$? wall $SECONDS s"; tail -c 1200 gpurun_out/bench_r02d.json; tail -3 gpurun_out/bench_r02d.err
