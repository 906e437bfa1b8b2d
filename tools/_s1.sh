set -x
timeout 900 python -m pytest tests/test_gpu_conv.py -x -q > gpurun_out/t_conv.log 2>&1; tail -5 gpurun_out/t_conv.log
timeout 900 python -m pytest tests/test_gpu_network.py -x -q -k "noscope or logits or real_extents" > gpurun_out/t_net.log 2>&1; tail -5 gpurun_out/t_net.log
for n in vgg16 resnet50 squeezenet1_0 shufflenet_v2_x1_0; do
  L=conv1; [ $n = vgg16 ] && L=features.0; [ $n = squeezenet1_0 ] && L=features.0
  for s in unprotected global-abft global-dot thread-one-sided; do timeout 300 python tools/ncu_netlayer.py $n 256 $s $L 1 2>&1 | grep "us "; done
done
bash tools/gpu_prof.sh dn_b resnet50 256 unprotected layer1.0.downsample,conv1
bash tools/gpu_prof.sh f2_b vgg16 256 unprotected features.2
