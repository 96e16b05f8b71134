python -m paper_2103_07329_b200.build > /dev/null
MRS_LIB=$PWD/paper_2103_07329_b200/libmrsolve_b200_checked.so timeout 900 python scripts/determinism_stress.py > gpurun_out/det_checked.log 2>&1; echo "checked rc=$?"; tail -9 gpurun_out/det_checked.log
timeout 900 python scripts/determinism_stress.py > gpurun_out/det.log 2>&1; echo "release rc=$?"; tail -3 gpurun_out/det.log
MRS_LIB=$PWD/paper_2103_07329_b200/libmrsolve_b200_checked.so timeout 1500 python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/pytest_checked.log 2>&1; echo "checked pytest rc=$?"; tail -3 gpurun_out/pytest_checked.log
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/pytest_kern.log 2>&1; echo "kernels rc=$?"; tail -3 gpurun_out/pytest_kern.log
