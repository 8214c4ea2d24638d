timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
PROBE_ORDERS=2 timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_flux --launch-skip 3 --launch-count 1 -o gpurun_out/flux_full -f python scripts/probe_perf.py 2000 > gpurun_out/ncu_flux.log 2>&1
PROBE_ORDERS=2 timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_sweep --launch-skip 6 --launch-count 1 -o gpurun_out/sweep_full -f python scripts/probe_perf.py 2000 > gpurun_out/ncu_sweep.log 2>&1
PROBE_ORDERS=2,1 timeout 300 python scripts/probe_perf.py 400 2000 3163 > gpurun_out/probe.txt 2>&1
cat gpurun_out/pytest_gpu.txt gpurun_out/probe.txt; tail -3 gpurun_out/ncu_flux.log
