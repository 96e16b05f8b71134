R=$PWD
python -m paper_2103_07329_b200.build > /dev/null
for rep in 1 2; do
for d in ab/7028b62 .; do for at in 0 1; do
  for c in c2 c3 c4; do
  (cd $R/$d && MRS_SPMM_AUTOTUNE=$at python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-spmm 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$d $c at=$at', $rep, round(d['ms_per_step'],3), round(d['roofline']['us_per_launch'],2), round(d['roofline']['us_per_launch_isolated'],2))")
  done
done; done; done
