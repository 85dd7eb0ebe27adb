#!/bin/bash
# One bench line per BASELINE config on the current box (round-2 results table):
#   tools/bench_all.sh > gpurun_out/r02_bench_all_configs.jsonl
cd "$(dirname "$0")/.." || exit 1
python bench.py -B 32 --batch 64 --steps 20 --warmup 5 2>/dev/null | tail -1
python bench.py -B 128 --steps 20 --warmup 5 2>/dev/null | tail -1
python bench.py -B 256 --steps 20 --warmup 5 2>/dev/null | tail -1
python bench.py -B 512 --steps 20 --warmup 5 2>/dev/null | tail -1
