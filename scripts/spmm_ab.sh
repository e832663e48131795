#!/usr/bin/env bash
python scripts/syev_ab.py
GCG_SYEV=batched python scripts/syev_ab.py
