#!/usr/bin/env bash
python scripts/kbench.py 2 2>&1 | grep -E "syev|svqb"
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
