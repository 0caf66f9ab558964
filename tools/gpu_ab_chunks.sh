#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
for cfgs in "1 2 1" "2 2 1" "4 2 1" "8 2 1" "4 3 1" "4 2 2" "8 2 2" "4 1 2" "16 2 1"; do
  set -- $cfgs
  echo -n "chunks=$1 schur_cap=$2 inv_cap=$3: "
  IRK_FACTOR_CHUNKS=$1 IRK_SCHUR_CAP=$2 IRK_INV_CAP=$3 python tools/time_factor.py 1 color | tail -1
done
