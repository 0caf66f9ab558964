#!/bin/bash
# A/B of the Schur-phase variants (IRK_SCHUR_MODE): factor parity tests, then factor timings
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" || exit 1
for m in ${MODES:-2 0}; do
  echo "== IRK_SCHUR_MODE=$m"
  IRK_SCHUR_MODE=$m timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "${TESTS:-inverse or factor or ilu0 or singular or golden or fullsize or implicit or refactor}" 2>&1 | tail -2
  for c in ${CFGS:-1}; do
  IRK_SCHUR_MODE=$m python tools/time_factor.py $c color ${NARG}
  IRK_SCHUR_MODE=$m timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_inverse_tc|k_schur" --csv --log-file $O/ab_schur_$m.csv python tools/time_factor.py $c color ${NARG} > /dev/null 2>&1
  python - <<PY
import csv,collections
rows=list(csv.reader(open("$O/ab_schur_$m.csv")))
hi=[i for i,r in enumerate(rows) if "Kernel Name" in r][0]; h=rows[hi]
k,v,u=h.index("Kernel Name"),h.index("Metric Value"),h.index("Metric Unit")
agg=collections.OrderedDict()
for r in rows[hi+1:]:
    x=float(r[v].replace(",","")); x*= {"ns":1e-3,"us":1.0,"ms":1e3,"nsecond":1e-3,"usecond":1.0,"msecond":1e3}.get(r[u],1.0)
    agg.setdefault(r[k].split("(")[0],[]).append(x)
for n,l in agg.items(): print("  ", n, "n=%d last4 mean %.1f us"%(len(l), sum(l[-4:])/len(l[-4:])))
PY
  done
done
