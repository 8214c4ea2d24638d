# ncu --set full captures of the iteration's kernels at 10M points (run under
# gpurun; reports land in gpurun_out/, summarised into profiles/ by
# scripts/ncu_summary.py and scripts/sass_mix.py).
#   bash scripts/ncu_kernels.sh <tag> [kernel-regex ...]
tag=${1:-r02}
shift
kernels=${@:-"k_flux_ws k_sweep_tile k_update"}
mkdir -p gpurun_out
export PROBE_NACA=4000x2500 PROBE_ORDERS=2
for k in $kernels; do
  skip=3
  [ "$k" = "k_sweep2" ] && skip=6
  [ "$k" = "k_sweep_tile" ] && skip=6
  timeout 400 ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip $skip --launch-count 1 \
      -o gpurun_out/${tag}_${k}10m -f python scripts/probe_perf.py > gpurun_out/${tag}_${k}.log 2>&1
  tail -2 gpurun_out/${tag}_${k}.log
done
