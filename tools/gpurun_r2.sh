timeout 900 python -m pytest tests/test_rls.py -q -x -v 2>&1 | grep -E "PASS|FAIL|Error|error|passed|failed" | head -20
