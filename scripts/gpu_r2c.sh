python -m paper_2103_07329_b200.build
timeout 900 python -m pytest tests/test_gpu_loopback.py tests/test_gpu_team.py -x -q > gpurun_out/pytest_team.log 2>&1; echo "team rc=$?"
tail -30 gpurun_out/pytest_team.log
