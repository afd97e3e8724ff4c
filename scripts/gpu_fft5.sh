for a in "c2 fft 32" "c3 fft 32" "c5 fft 64"; do python scripts/bench_products.py $a 3 2>&1 | tail -2; done
