python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_inverse_tc" -c 1 -f -o /tmp/inv_tc python tools/time_factor.py 1 color > /dev/null 2>&1
ncu -i /tmp/inv_tc.ncu-rep --page raw --csv > gpurun_out/inv_tc2_raw.csv 2>/dev/null
ncu -i /tmp/inv_tc.ncu-rep --page source --csv --print-source sass > gpurun_out/inv_tc2_src.csv 2>/dev/null
