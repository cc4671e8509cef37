python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q 2>&1 | grep -E "passed|failed|Error|^E " | head -20
