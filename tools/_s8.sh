timeout 900 python -m pytest tests/test_gpu_conv.py -x -q > gpurun_out/t_8.log 2>&1; tail -2 gpurun_out/t_8.log
timeout 900 python -m pytest tests/test_gpu_network.py tests/test_gpu_dlrm.py tests/test_gpu_chain.py -x -q > gpurun_out/t_8n.log 2>&1; tail -2 gpurun_out/t_8n.log
for n in vgg16 resnet50 squeezenet1_0 shufflenet_v2_x1_0; do
  L=conv1; [ $n = vgg16 ] && L=features.0; [ $n = squeezenet1_0 ] && L=features.0
  for s in unprotected global-abft; do timeout 300 python tools/ncu_netlayer.py $n 256 $s $L 1 2>&1 | grep "us " | cut -c1-80; done
done
timeout 300 python tools/ncu_netlayer.py vgg16 256 global-abft features.10,features.12,features.14,features.17,features.19,features.24,features.28,classifier.0 1 2>&1 | grep "us " | cut -c1-80
timeout 300 python tools/ncu_netlayer.py vgg16 256 global-abft features.10,features.12,features.14,features.17,features.19,features.24,features.28,classifier.0 1 32 2>&1 | grep "us " | cut -c1-80
timeout 300 python tools/ncu_netlayer.py vgg16 256 unprotected features.10,features.12,features.14,features.17,features.19,features.24,features.28,classifier.0 1 2>&1 | grep "us " | cut -c1-80
