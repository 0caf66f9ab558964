#!/bin/bash
# One GPU round: gpu tests, bench, launch list, --set full capture of the top kernels.
# usage (via gpurun): bash tools/gpu_round.sh TAG [skip-tests]
TAG=${1:-r1}
O=gpurun_out
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build_$TAG.log 2>&1 || { echo build failed; tail -30 $O/build_$TAG.log; exit 1; }
if [ "$2" != "skip-tests" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu_$TAG.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke_$TAG.log
fi
timeout 900 python bench.py > $O/bench_$TAG.log 2>&1; echo "bench rc=$?"; tail -1 $O/bench_$TAG.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file $O/launches_$TAG.csv python bench.py --steps 1 --warmup 1 --profile --no-alt --jnorm 2.4496432463318416 \
  > $O/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
# full capture of the hot kernels of one timed step (launches after warmup)
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"k_schur|k_inverse|k_unc|k_stage_matvec|k_multidot|k_update|k_finish" \
  --profile-from-start off -c ${NCU_COUNT:-12} -f -o /tmp/full_$TAG \
  python bench.py --steps 1 --warmup 1 --profile --no-alt --jnorm 2.4496432463318416 > $O/ncu_full_$TAG.log 2>&1
echo "ncu full rc=$?"
ncu -i /tmp/full_$TAG.ncu-rep --page raw --csv > $O/raw_$TAG.csv 2>/dev/null
ls -la $O
