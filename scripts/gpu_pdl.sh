python -m paper_2103_07329_b200.build > /dev/null
for rep in 1 2; do for pdl in 0 1; do for c in c2 c1 c3; do
  MRS_PDL=$pdl python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-spmm 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c pdl=$pdl', $rep, round(d['ms_per_step'],3), d['config']['iterations'], d['details']['kernels_per_iteration'])"
done; done; done
