# One GPU round-trip of the build -> measure loop (run under gpurun):
#   GPU tests, per-size device timing, ncu --set full of the flux kernel.
#   TAG names the outputs; SIZES the probe clouds.
TAG=${TAG:-it}
SIZES=${SIZES:-400 2000 3163}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/${TAG}_pytest.txt
PROBE_ORDERS=2,1 timeout 600 python scripts/probe_perf.py $SIZES > gpurun_out/${TAG}_probe.txt 2>&1
if [ -n "$NCU" ]; then
  PROBE_ORDERS=2 timeout 300 ncu --set full --import-source on --clock-control none -k regex:${NCU} --launch-skip 3 --launch-count 1 -o gpurun_out/${TAG}_ncu -f python scripts/probe_perf.py 2000 > gpurun_out/${TAG}_ncu.log 2>&1
fi
cat gpurun_out/${TAG}_pytest.txt gpurun_out/${TAG}_probe.txt
