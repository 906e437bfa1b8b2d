timeout 900 python -m pytest tests/test_gpu_conv.py -x -q > gpurun_out/t_conv4.log 2>&1; tail -3 gpurun_out/t_conv4.log
for n in vgg16 resnet50 squeezenet1_0 shufflenet_v2_x1_0; do
  L=conv1; [ $n = vgg16 ] && L=features.0; [ $n = squeezenet1_0 ] && L=features.0
  for s in unprotected global-abft thread-one-sided; do timeout 300 python tools/ncu_netlayer.py $n 256 $s $L 1 2>&1 | grep "us " | cut -c1-80; done
  timeout 300 python tools/ncu_netlayer.py $n 256 unprotected $L 1 8 2>&1 | grep "us " | cut -c1-80
done
for f in 0 8; do
timeout 300 python tools/ncu_netlayer.py vgg16 256 unprotected features.2,features.5,features.7,features.14 1 $f 2>&1 | grep "us " | cut -c1-80
timeout 300 python tools/ncu_netlayer.py resnet50 256 unprotected layer1.0.conv3,layer1.0.downsample,layer2.0.conv3,layer1.0.conv2,layer1.0.conv1 1 $f 2>&1 | grep "us " | cut -c1-80
done
bash tools/gpu_prof.sh c1_e resnet50 256 unprotected conv1
bash tools/gpu_prof.sh f2_e vgg16 256 unprotected features.2
