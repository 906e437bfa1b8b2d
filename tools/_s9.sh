timeout 900 python -m pytest tests/test_gpu_conv.py -x -q -k "tail_split or copy_depths or stem or exact_int" > gpurun_out/t_9.log 2>&1; tail -3 gpurun_out/t_9.log
for d in 0 128 320; do
for n in vgg16 resnet50 squeezenet1_0; do
  L=conv1; [ $n = vgg16 ] && L=features.0; [ $n = squeezenet1_0 ] && L=features.0
  timeout 300 python tools/ncu_netlayer.py $n 256 unprotected $L 1 $d 2>&1 | grep "us " | cut -c1-70
done
done
timeout 600 python tools/store_probe.py 2>&1 | tail -30
