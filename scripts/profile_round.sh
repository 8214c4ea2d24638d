# Round-end measurement (run under gpurun; outputs in gpurun_out/, summarised
# into profiles/ by scripts/ncu_summary.py and scripts/sass_mix.py):
#   bash scripts/profile_round.sh <tag>
# - the bench line (N=1, default workload) and the reference arm
# - ncu --set full of the flux, sweep and update kernels at 10M points
# - the ncu launch list of a short bench run (per-launch device times)
tag=${1:-r02}
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/${tag}_bench_reference.json 2> gpurun_out/${tag}_bench_reference.err
bash scripts/ncu_kernels.sh ${tag} k_flux_ws k_sweep_tile k_update
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-sizes \
    --no-e2e > gpurun_out/${tag}_b_ncu.log 2>&1
tail -c 400 gpurun_out/${tag}_bench.json; tail -c 300 gpurun_out/${tag}_bench_reference.json; tail -3 gpurun_out/${tag}_bench.err
