python -m paper_2103_07329_b200.build
timeout 900 python scripts/spmm_variants.py > gpurun_out/spmm_variants2.json 2> gpurun_out/spmm_variants2.err; echo "variants rc=$?"
