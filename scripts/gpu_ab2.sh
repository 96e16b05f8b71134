R=$PWD
python -m paper_2103_07329_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_loopback.py tests/test_gpu_team.py tests/test_gpu_vec32.py -x -q > gpurun_out/pytest_lt.log 2>&1; echo "team rc=$?"; tail -3 gpurun_out/pytest_lt.log
for d in ab/7028b62 .; do
  cd $R/$d; for gm in "128 16" "128 8" "64 8"; do echo "$d $(MRS_SPMM_AUTOTUNE=0 python scripts/p7_time.py $gm)"; done
done
cd $R
for d in ab/7028b62 .; do for at in 0 1; do
  for c in c2 c3 c4; do
  (cd $R/$d && MRS_SPMM_AUTOTUNE=$at python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-spmm 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$d $c at=$at', round(d['ms_per_step'],3), round(d['roofline']['us_per_launch'],2), round(d['roofline']['us_per_launch_isolated'],2))")
  done
done; done
