#!/bin/bash
# config-3 multi-RHS apply: knob sweep per block size (each setting in its own process: knobs are read once)
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" || exit 1
: > $O/tune_cfg3.log
for nb in ${NBS:-24 40}; do
 for knobs in "" "IRK_SEG_NST=3" "IRK_SEG_NST=4" "IRK_APPLY_WSG=2" "IRK_APPLY_WSG=2 IRK_SEG_NST=3" "IRK_APPLY_SEG=0" "IRK_APPLY_SEG=0 IRK_APPLY_CTAS=6" "IRK_APPLY_SEG=0 IRK_APPLY_CTAS=8" "IRK_PDL=0"; do
  echo "== nb=$nb $knobs" >> $O/tune_cfg3.log
  env $knobs timeout 300 python tools/sweep.py config3 --nb $nb --s ${SS:-3 4} 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('   s=%d apply %.4f ms frac %.3f matvec frac %.3f refactor %.2f ms'%(d['s'],d['apply_ms'],d['apply_frac'],d['matvec_frac'],d['refactor_ms']))
" >> $O/tune_cfg3.log
 done
done
cat $O/tune_cfg3.log
