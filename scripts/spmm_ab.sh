#!/usr/bin/env bash
for v in 2 4; do for o in 0 1; do GCG_SPMM_VEC=$v GCG_SPMM_ORDER=$o python scripts/spmm_ab.py 2 3; done; done
