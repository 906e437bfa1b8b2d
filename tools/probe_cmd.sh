timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_final.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_final.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
bash tools/profile_round.sh r01d
timeout 2400 python tools/netbench.py --nets resnet50,vgg16,alexnet,squeezenet1_0,shufflenet_v2_x1_0,densenet161,resnext50_32x4d,wide_resnet50_2 --configs hd1,b64,b256 --cudnn --out gpurun_out/netbench_final.jsonl > gpurun_out/netbench_final.log 2>&1
python tools/gemm_sweep.py > gpurun_out/gemm_sweep_final.log 2>&1
python tools/scheme_study.py --out gpurun_out/scheme_study_final.jsonl > gpurun_out/scheme_study_final.log 2>&1
