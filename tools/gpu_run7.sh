python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
python tools/time_factor.py 1 color; IRK_INV_TC=0 python tools/time_factor.py 1 color
python tools/time_factor.py 2 color 16; IRK_INV_TC=0 python tools/time_factor.py 2 color 16
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/fac_c1_tc.csv -k regex:"k_inverse|k_schur" python tools/time_factor.py 1 color > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_s7.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu_s7.log
