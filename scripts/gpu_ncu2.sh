R=$PWD
python -m paper_2103_07329_b200.build > /dev/null
for d in ab/7028b62 .; do
  cd $R/$d
  tag=$(basename $d)
  MRS_SPMM_AUTOTUNE=0 python scripts/ncu_p7.py 128 16 > /tmp/plain_$tag.log 2>&1 || { echo plain fail; cat /tmp/plain_$tag.log; }
  MRS_SPMM_AUTOTUNE=0 ncu --set full --clock-control none -k regex:spmm_kernel -s 2 -c 1 -o /tmp/p7_$tag python scripts/ncu_p7.py 128 16 > /tmp/ncu_$tag.log 2>&1; echo "ncu $tag rc=$?"
  ncu -i /tmp/p7_$tag.ncu-rep --page details --csv > $R/gpurun_out/p7_m16_${tag}_details.csv 2>&1
  ncu -i /tmp/p7_$tag.ncu-rep --page raw --csv > $R/gpurun_out/p7_m16_${tag}_raw.csv 2>&1
done
