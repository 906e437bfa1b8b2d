python bench.py > gpurun_out/bench_r01m.json 2>gpurun_out/bench_r01m.err
