BENCH_SHARE_GPU=1 BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-secondary --nets squeezenet1_0,resnet50 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
echo "rc=$?"; tail -c 800 gpurun_out/bench_n2.json; grep -iE "error|Traceback" gpurun_out/bench_n2.err | head -5
timeout 600 python bench.py --impl reference --gpus 2 --steps 1 --warmup 1 | head -c 300
