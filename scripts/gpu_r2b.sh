python -m paper_2103_07329_b200.build
timeout 900 python -m pytest tests/test_gpu_loopback.py -x -q > gpurun_out/pytest_loop.log 2>&1; echo "loop rc=$?"
tail -30 gpurun_out/pytest_loop.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r2b.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_r2b.log
python bench.py --steps 10 --warmup 3 --no-cpu --quick > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err; echo "bench rc=$?"
