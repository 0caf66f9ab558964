#!/bin/bash
# A/B of the tensor-core inverse variants: parity tests, then factor timings (events + per-kernel ncu durations)
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "inverse or factor or ilu0 or singular or golden" 2>&1 | tail -4
for bg in ${BGS:-2 1}; do
  echo "== IRK_INV_BG=$bg"; IRK_INV_BG=$bg python tools/time_factor.py 1 color
  IRK_INV_BG=$bg timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_inverse|k_schur" --csv --log-file $O/ab_inv_bg$bg.csv python tools/time_factor.py 1 color > /dev/null 2>&1
  python - <<PY
import csv,collections
rows=list(csv.reader(open("$O/ab_inv_bg$bg.csv")))
hi=[i for i,r in enumerate(rows) if "Kernel Name" in r][0]; h=rows[hi]
k,v=h.index("Kernel Name"),h.index("Metric Value")
agg=collections.OrderedDict()
for r in rows[hi+1:]:
    agg.setdefault(r[k].split("(")[0],[]).append(float(r[v].replace(",","")))
for n,l in agg.items(): print(n, "n=%d last4 mean %.1f us"%(len(l), sum(l[-4:])/len(l[-4:])/1e3 if max(l)>1e4 else sum(l[-4:])/len(l[-4:])))
PY
done
