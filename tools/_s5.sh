for m in 2 3; do
for n in vgg16 resnet50 squeezenet1_0 shufflenet_v2_x1_0; do
  L=conv1; [ $n = vgg16 ] && L=features.0; [ $n = squeezenet1_0 ] && L=features.0
  ABFT_CONV_MODE=$m timeout 300 python tools/ncu_netlayer.py $n 256 unprotected $L 1 2>&1 | grep "us " | cut -c1-80
done
done
