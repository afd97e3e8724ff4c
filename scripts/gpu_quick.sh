#!/bin/bash
# Quick product check on one B200: product parity tests, then block-product timings on c5 / c3 / c2.
# Usage: bash scripts/gpu_quick.sh <tag> [pytest -k expression]
tag=${1:-quick}; out=gpurun_out/$tag; mkdir -p $out
kexpr=${2:-products}
timeout 900 python -m pytest tests -m gpu -q -x -k "$kexpr" --timeout 600 > $out/pytest.log 2>&1; tail -2 $out/pytest.log
for c in c5 c3 c2; do timeout 300 python scripts/prof_products.py $c fft 2>&1 | tail -2; done
