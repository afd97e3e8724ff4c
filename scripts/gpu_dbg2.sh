for c in c2 c3; do for i in 1 2; do SSA_DEBUG=1 python scripts/debug_decompose.py $c auto 2>&1 | grep -E "host ms|^c[0-9]" ; done; done
for c in c2; do SSA_ORTH_FAST=1 SSA_DEBUG=1 python scripts/debug_decompose.py $c auto 2>&1 | grep -E "host ms|^c[0-9]" ; done
timeout 300 python scripts/bench_products.py c2 tc 32 20
