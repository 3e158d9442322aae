timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -6
timeout 2400 python tools/config_runs.py c4 c3 c5 2>&1 | grep -E "^c[345]|Error|error" | cut -c1-1200
