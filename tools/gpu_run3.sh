set -x
free -g | head -2
nproc
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_s4.log 2>&1 || { tail -20 gpurun_out/build_s4.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_s4.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu_s4.log
timeout 900 python tools/sweep.py config3 > gpurun_out/sweep_c3.jsonl 2> gpurun_out/sweep_c3.err; echo "c3 rc=$?"; tail -3 gpurun_out/sweep_c3.err
timeout 900 python tools/sweep.py config4 > gpurun_out/sweep_c4.jsonl 2> gpurun_out/sweep_c4.err; echo "c4 rc=$?"; tail -3 gpurun_out/sweep_c4.err
timeout 1200 python tools/sweep.py config2kernels > gpurun_out/sweep_c2.jsonl 2> gpurun_out/sweep_c2.err; echo "c2 rc=$?"; tail -3 gpurun_out/sweep_c2.err
timeout 600 python bench.py --no-alt > gpurun_out/bench_s4.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_s4.log | cut -c1-300
