mkdir -p gpurun_out
for sch in unprotected global-fused; do
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -c 1 -k regex:abft_gemm -o /tmp/p_$sch -f python tools/ncu_netlayer.py vgg16 256 $sch features.19 1 6144 > gpurun_out/s45_log_$sch.txt 2>&1
python tools/ncu_layer_summary.py /tmp/p_$sch.ncu-rep "vgg16 features.19 $sch pair" > gpurun_out/s45_summary_$sch.txt 2>&1
python tools/ncu_stalls.py /tmp/p_$sch.ncu-rep > gpurun_out/s45_stalls_$sch.txt 2>&1
done
