python -m paper_2103_07329_b200.build
timeout 900 python scripts/spmm_variants.py > gpurun_out/spmm_variants.json 2> gpurun_out/spmm_variants.err; echo "variants rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r2d.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_r2d.log
python bench.py --steps 10 --warmup 3 --no-cpu --quick > gpurun_out/bench_r2d.json 2> gpurun_out/bench_r2d.err; echo "bench rc=$?"
