python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 120 python tools/t2sm_check.py; echo check=$?
