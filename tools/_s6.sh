timeout 900 python -m pytest tests/test_gpu_conv.py tests/test_gpu_parity.py tests/test_gpu_chain.py -x -q > gpurun_out/t_6.log 2>&1; tail -3 gpurun_out/t_6.log
for n in vgg16 resnet50 squeezenet1_0 shufflenet_v2_x1_0; do
  L=conv1; [ $n = vgg16 ] && L=features.0; [ $n = squeezenet1_0 ] && L=features.0
  for s in unprotected global-abft thread-one-sided; do timeout 300 python tools/ncu_netlayer.py $n 256 $s $L 1 2>&1 | grep "us " | cut -c1-80; done
done
for f in 0 16; do
timeout 300 python tools/ncu_netlayer.py vgg16 256 unprotected features.2,features.5,features.7 1 $f 2>&1 | grep "us " | cut -c1-80
timeout 300 python tools/ncu_netlayer.py resnet50 256 unprotected layer1.0.conv2,layer1.0.conv1,layer2.0.conv1,layer2.1.conv2 1 $f 2>&1 | grep "us " | cut -c1-80
timeout 300 python tools/ncu_netlayer.py squeezenet1_0 256 unprotected features.3.squeeze,features.3.expand1x1,features.3.expand3x3,features.5.expand3x3 1 $f 2>&1 | grep "us " | cut -c1-80
done
timeout 900 python -m pytest tests/test_gpu_network.py -x -q > gpurun_out/t_6n.log 2>&1; tail -3 gpurun_out/t_6n.log
