mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_naca.py -m gpu -q -x 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_naca.json 2> gpurun_out/bench_naca.err
timeout 600 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_naca_ref.json 2>> gpurun_out/bench_naca.err
cat gpurun_out/bench_naca.json gpurun_out/bench_naca_ref.json; tail -3 gpurun_out/bench_naca.err
