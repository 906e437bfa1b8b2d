timeout 900 python -m pytest tests/test_gpu_conv.py -x -q > gpurun_out/t_7.log 2>&1; tail -2 gpurun_out/t_7.log
for n in vgg16 resnet50 squeezenet1_0 shufflenet_v2_x1_0; do
  L=conv1; [ $n = vgg16 ] && L=features.0; [ $n = squeezenet1_0 ] && L=features.0
  for s in unprotected global-abft thread-one-sided; do timeout 300 python tools/ncu_netlayer.py $n 256 $s $L 1 2>&1 | grep "us " | cut -c1-80; done
done
bash tools/gpu_prof.sh c1_f resnet50 256 unprotected conv1
