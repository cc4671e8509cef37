python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 500 python -m pytest tests/test_gpu_parity.py -x -q -k "npr" 2>&1 | grep -E "passed|failed|^E " | head -12
