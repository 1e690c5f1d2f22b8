#!/bin/bash
# quick GPU regression: parity subset + bench line
python -m pytest tests -q -m gpu -x -k "random_vs_oracle or edge or strided or empty or kmax or errors or large_block or generators or properties" 2>&1 | tail -3
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1
