# Round-end measurement: bench line + ncu --set full of the flux, sweep and update kernels at
# 10M points + the ncu launch list of a short bench (run under gpurun; outputs in gpurun_out/,
# summarised into profiles/ by scripts/ncu_summary.py and scripts/sass_mix.py).
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
export PROBE_NACA=4000x2500 PROBE_ORDERS=2
timeout 400 ncu --set full --import-source on --clock-control none -k regex:k_flux_ws --launch-skip 3 --launch-count 1 -o gpurun_out/r01f_flux10m -f python scripts/probe_perf.py > gpurun_out/ncu1.log 2>&1
timeout 400 ncu --set full --import-source on --clock-control none -k regex:k_sweep --launch-skip 6 --launch-count 1 -o gpurun_out/r01f_sweep10m -f python scripts/probe_perf.py > gpurun_out/ncu2.log 2>&1
timeout 400 ncu --set full --import-source on --clock-control none -k regex:k_update --launch-skip 3 --launch-count 1 -o gpurun_out/r01f_update10m -f python scripts/probe_perf.py > gpurun_out/ncu3.log 2>&1
unset PROBE_NACA
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01f_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-steady --large-naca 0 > gpurun_out/b_ncu.log 2>&1
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err; tail -2 gpurun_out/ncu1.log
