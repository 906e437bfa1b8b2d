for kp in 0 1; do
ABFT_KPAIR=$kp python tools/probe.py "50176 64 576 unprotected 0" "50176 64 576 unprotected 64" "50176 64 576 thread-one-sided 0 0 aug" "50176 64 576 global-abft 0 0 gck" "8192 8192 8192 global-abft 0 0 gck"
done > gpurun_out/probe_5k.log 2>&1
