python -m paper_2103_07329_b200.build
timeout 900 python -m pytest tests/test_gpu_vec32.py -x -q > gpurun_out/pytest_vec32.log 2>&1; echo "vec32 rc=$?"
tail -5 gpurun_out/pytest_vec32.log
for c in c2 c2v32 c3 c3v32; do
python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-spmm > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
done
python scripts/warm_profile.py --config c2 > gpurun_out/warm_c2.txt 2>&1
python scripts/warm_profile.py --config c3 > gpurun_out/warm_c3.txt 2>&1
python scripts/warm_profile.py --config c3v32 > gpurun_out/warm_c3v32.txt 2>&1
