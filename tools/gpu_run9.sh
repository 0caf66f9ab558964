python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
NSTS=2,3,4,6 TUNE_G=1,2,3,4,5 python tools/tune_apply.py 2>&1 | tail -25
