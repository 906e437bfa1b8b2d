timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/t_20.log 2>&1; tail -3 gpurun_out/t_20.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash tools/r02_profiles.sh r02
