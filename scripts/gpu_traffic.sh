for a in "c2 fft 32" "c3 fft 32" "c4 fft 32" "c1 direct 16"; do
  set -- $a
  python scripts/traffic_products.py $1 $2 $3 > /dev/null 2>&1 && ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file gpurun_out/traffic_$1_$2.csv python scripts/traffic_products.py $1 $2 $3 > /dev/null 2>&1; echo "$a $?"
done
