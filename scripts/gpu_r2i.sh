python -m paper_2103_07329_b200.build
for at in 0 1; do for c in c2 c3 c4; do
MRS_SPMM_AUTOTUNE=$at python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-spmm > gpurun_out/ab_${c}_$at.json 2> gpurun_out/ab_${c}_$at.err; echo "bench $c at=$at rc=$?"
done; done
MRS_SPMM_AUTOTUNE=0 python scripts/warm_profile.py --config c2 > gpurun_out/warm_c2_at0.txt 2>&1
