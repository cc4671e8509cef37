python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "out_of_core" 2>&1 | grep -E "Error|error|assert|^E " | head -30
