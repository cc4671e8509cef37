python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -s -k "config3" 2>&1 | grep -E "config 3|passed|failed|^E " | head -10
free -g | head -2
