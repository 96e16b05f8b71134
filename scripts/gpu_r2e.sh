python -m paper_2103_07329_b200.build
python scripts/ncu_c5.py 8 1 > gpurun_out/ncu_c5_plain.log 2>&1 || exit 1
for cfg in "8 1 m8_lane" "8 2 m8_coop" "1 1 m1_lane"; do
  set -- $cfg
  ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -s 1 -c 1 -o /tmp/c5_$3 python scripts/ncu_c5.py $1 $2 > /tmp/ncu_$3.log 2>&1; echo "ncu $3 rc=$?"
  ncu -i /tmp/c5_$3.ncu-rep --page details --csv > gpurun_out/c5_$3_details.csv 2>&1
  ncu -i /tmp/c5_$3.ncu-rep --page raw --csv > gpurun_out/c5_$3_raw.csv 2>&1
  ncu -i /tmp/c5_$3.ncu-rep --page source --csv --print-source sass > /tmp/c5_$3_src.csv 2>&1
  head -c 3000000 /tmp/c5_$3_src.csv > gpurun_out/c5_$3_src.csv
done
ls -la gpurun_out
