mkdir -p gpurun_out
for sch in unprotected; do
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -c 1 -o /tmp/p_c12 -f python tools/ncu_netlayer.py vgg16 256 $sch features.2 1 > gpurun_out/s36_log.txt 2>&1
python tools/ncu_stalls.py /tmp/p_c12.ncu-rep > gpurun_out/s36_stalls.txt 2>&1
STALL_ORDER=1 python tools/ncu_stalls.py /tmp/p_c12.ncu-rep 344064 >> gpurun_out/s36_stalls.txt 2>&1
python tools/ncu_layer_summary.py /tmp/p_c12.ncu-rep "vgg16 features.2 $sch" > gpurun_out/s36_summary.txt 2>&1
done
