#!/usr/bin/env bash
python scripts/kbench.py 2 2>&1 | grep -E "CG|cg_|spmm "
timeout 600 python -m pytest tests -m gpu -q -x -k "cg or solver" 2>&1 | tail -2
