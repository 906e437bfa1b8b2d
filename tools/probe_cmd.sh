timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_r01s.log 2>&1; tail -2 gpurun_out/pytest_gpu_r01s.log
for S in "2048 512 512" "2048 512 16"; do
python tools/probe.py "$S unprotected 0" "$S global-abft 0" "$S global-abft 0 0 gck"
done > gpurun_out/probe_fl2.log 2>&1
python bench.py > gpurun_out/bench_r01s.json 2>gpurun_out/bench_r01s.err
