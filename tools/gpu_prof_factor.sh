#!/bin/bash
# ncu --set full of the factor kernels (tools/time_factor.py), raw + source pages -> gpurun_out/
# usage: bash tools/gpu_prof_factor.sh TAG "ENV=.. ENV2=.." [kernel-regex] [config] [ordering]
TAG=$1; ENVS=$2; RX=${3:-"k_inverse|k_schur"}; CFG=${4:-1}; ORD=${5:-color}
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" || exit 1
env $ENVS python tools/time_factor.py $CFG $ORD
env $ENVS timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$RX" --launch-skip ${SKIP:-6} -c ${COUNT:-3} -f -o /tmp/pf_$TAG python tools/time_factor.py $CFG $ORD > $O/pf_$TAG.log 2>&1
ncu -i /tmp/pf_$TAG.ncu-rep --page raw --csv > $O/pf_raw_$TAG.csv 2>/dev/null
ncu -i /tmp/pf_$TAG.ncu-rep --page source --csv --print-source sass > $O/pf_src_$TAG.csv 2>/dev/null
ls -la $O/pf_*_$TAG.csv
