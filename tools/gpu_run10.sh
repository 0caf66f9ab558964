python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_s10.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|Error|error" gpurun_out/pytest_gpu_s10.log | tail -8
python tools/sweep.py config0; IRK_CPL_GENERIC=1 python tools/sweep.py config0
python tools/sweep.py config4 --dtn 100 --jnorm 2.4496432463318416; IRK_CPL_GENERIC=1 python tools/sweep.py config4 --dtn 100 --jnorm 2.4496432463318416
