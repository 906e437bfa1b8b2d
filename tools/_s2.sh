timeout 900 python -m pytest tests/test_gpu_conv.py -x -q > gpurun_out/t_conv2.log 2>&1; tail -3 gpurun_out/t_conv2.log
for n in vgg16 resnet50 squeezenet1_0 shufflenet_v2_x1_0; do
  L=conv1; [ $n = vgg16 ] && L=features.0; [ $n = squeezenet1_0 ] && L=features.0
  for s in unprotected global-abft thread-one-sided; do timeout 300 python tools/ncu_netlayer.py $n 256 $s $L 1 2>&1 | grep "us " | cut -c1-90; done
done
timeout 300 python tools/ncu_netlayer.py resnet50 256 unprotected layer1.0.conv3,layer1.1.conv3,layer2.0.conv3,layer1.0.downsample 1 2>&1 | grep "us " | cut -c1-90
timeout 300 python tools/ncu_netlayer.py resnet50 256 thread-one-sided layer1.0.conv3,layer2.0.conv3 1 2>&1 | grep "us " | cut -c1-90
bash tools/gpu_prof.sh c1_c resnet50 256 unprotected conv1
bash tools/gpu_prof.sh ds_c resnet50 256 unprotected layer1.0.downsample
