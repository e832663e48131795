#!/usr/bin/env bash
python scripts/kbench.py 2 2>&1 | grep -E "syev|svqb"
timeout 600 python -m pytest tests -m gpu -q -x -k "syev or svqb or solver" 2>&1 | tail -3
