timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/t_10.log 2>&1; tail -3 gpurun_out/t_10.log
timeout 600 python tools/store_probe.py 2>&1 | grep -v torch | tail -20
for f in 0 512; do
for n in vgg16 resnet50 squeezenet1_0 shufflenet_v2_x1_0; do
  L=conv1; [ $n = vgg16 ] && L=features.0; [ $n = squeezenet1_0 ] && L=features.0
  timeout 300 python tools/ncu_netlayer.py $n 256 unprotected $L 1 $f 2>&1 | grep "us " | cut -c1-70
done
timeout 300 python tools/ncu_netlayer.py resnet50 256 unprotected layer1.0.conv3,layer1.0.downsample,layer2.0.conv3,layer1.0.conv2 1 $f 2>&1 | grep "us " | cut -c1-70
timeout 300 python tools/ncu_netlayer.py vgg16 256 unprotected features.2,features.5,features.7,features.12 1 $f 2>&1 | grep "us " | cut -c1-70
done
