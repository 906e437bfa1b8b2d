timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_r01q.log 2>&1; tail -2 gpurun_out/pytest_gpu_r01q.log
python tools/gemm_sweep.py --stamps --only-stamps > gpurun_out/stamps6.log 2>&1
python tools/probe.py "2048 512 512 unprotected 64" "128 64 512 unprotected 64" "128 64 32768 unprotected 64" "2048 512 16 unprotected 0" "4096 4096 4096 unprotected 0" > gpurun_out/probe_lv.log 2>&1
python tools/chain_probe2.py > gpurun_out/chain_probe7.log 2>&1
python bench.py > gpurun_out/bench_r01q.json 2>gpurun_out/bench_r01q.err
