#!/bin/bash
# quick GPU iteration: tests matching $1 (pytest -k), then bench with extra args $2
K="$1"; shift
timeout 900 python -m pytest tests -m gpu -q -x -k "$K" 2>&1 | tail -15
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" 2>&1 | tail -2
