SECONDS=0; timeout 1500 python bench.py --details gpurun_out/bench_details_r02c.json > gpurun_out/bench_r02c.json 2> gpurun_out/bench_r02c.err
echo "bench rc=$? wall $SECONDS s"; tail -c 1500 gpurun_out/bench_r02c.json; tail -3 gpurun_out/bench_r02c.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r02c.json 2>&1; tail -c 300 gpurun_out/bench_ref_r02c.json
timeout 1500 ncu --nvtx --nvtx-include "timed_ig/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r02c.csv python bench.py --steps 1 --warmup 3 --no-secondary > gpurun_out/bench_ncu_r02c.log 2>&1
echo "ncu rc=$?"; wc -l gpurun_out/launches_r02c.csv
