TACOS_CLUSTER=4 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | grep -v "^\s*$" | grep -E "FAILED|Error|error|assert|test_" | head -20
git stash list >/dev/null 2>&1
