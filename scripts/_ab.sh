for v in "LSKUM_SWEEP_BLOCK=256" "LSKUM_SWEEP_BLOCK=128"; do
  echo "== $v"; env $v PROBE_ORDERS=2 timeout 300 python scripts/probe_perf.py 400 3163 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: print(l.strip()); continue
  k={a:b for a,b,c in d['kernels']}; print(d['n'], round(d['ms_per_it'],4), 'sweep', k.get('q_derivatives'), 'flux', k['flux_residual'])"
done
