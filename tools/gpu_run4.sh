python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_s5.log 2>&1 || { tail -20 gpurun_out/build_s5.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_s5.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu_s5.log
timeout 600 python bench.py --no-alt > gpurun_out/bench_s5.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_s5.log | cut -c1-200
timeout 900 python tools/sweep.py config2kernels --jnorm 2.5 > gpurun_out/sweep_c2.jsonl 2> gpurun_out/sweep_c2.err; echo "c2 rc=$?"; tail -3 gpurun_out/sweep_c2.err; cat gpurun_out/sweep_c2.jsonl
timeout 900 python tools/sweep.py config3 > gpurun_out/sweep_c3.jsonl 2> gpurun_out/sweep_c3.err; echo "c3 rc=$?"; tail -3 gpurun_out/sweep_c3.err
timeout 900 python tools/sweep.py config4 --jnorm 2.4496432463318416 > gpurun_out/sweep_c4.jsonl 2> gpurun_out/sweep_c4.err; echo "c4 rc=$?"; tail -3 gpurun_out/sweep_c4.err
