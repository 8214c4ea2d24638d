export PROBE_NACA=520x308,4000x2500 PROBE_ORDERS=2
echo "== with ktimer"; python scripts/probe_perf.py 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); print(d['n'], round(d['ms_per_it'],4))"
cp paper_2403_13287_b200/nokt/liblskum_b200.so paper_2403_13287_b200/liblskum_b200.so
echo "== no ktimer"; python scripts/probe_perf.py 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); print(d['n'], round(d['ms_per_it'],4))"
