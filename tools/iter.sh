#!/bin/bash
# usage: iter.sh tag  -- gpu tests + short bench (no e2e/cpu legs)
tag=$1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/${tag}_tests.log
timeout 600 python bench.py --no-e2e --no-cpu-baseline --out gpurun_out/${tag}_bench.jsonl > gpurun_out/${tag}_bench.log 2>&1; echo bench rc=$?
