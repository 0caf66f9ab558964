python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_s6.log 2>&1 || { tail -20 gpurun_out/build_s6.log; exit 1; }
python tools/time_factor.py 1 color; IRK_INV_TC=0 python tools/time_factor.py 1 color
python tools/time_factor.py 2 color 16; IRK_INV_TC=0 python tools/time_factor.py 2 color 16
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fac_c1_tc.csv python tools/time_factor.py 1 color > /dev/null 2>&1
IRK_INV_TC=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fac_c1_notc.csv python tools/time_factor.py 1 color > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fac_c2_tc.csv python tools/time_factor.py 2 color 16 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_inverse|k_schur" -c 8 -f -o gpurun_out/fac_full python tools/time_factor.py 1 color > /dev/null 2>&1
ncu -i gpurun_out/fac_full.ncu-rep --page raw --csv > gpurun_out/fac_full_raw.csv 2>/dev/null
ncu --set full --clock-control none --import-source on -k regex:"k_inverse|k_schur" -c 6 -f -o gpurun_out/fac2_full python tools/time_factor.py 2 color 16 > /dev/null 2>&1
ncu -i gpurun_out/fac2_full.ncu-rep --page raw --csv > gpurun_out/fac2_full_raw.csv 2>/dev/null
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_s6.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu_s6.log
