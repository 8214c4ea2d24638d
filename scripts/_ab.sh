export PROBE_NACA=520x308,4000x2500 PROBE_ORDERS=2
python scripts/probe_perf.py 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: print(l.strip()); continue
  k={a:b for a,b,c in d['kernels']}; print(d['n'], round(d['ms_per_it'],4), 'sweep', k.get('q_derivatives'), 'flux', k['flux_residual'])"
