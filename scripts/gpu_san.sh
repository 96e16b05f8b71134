TOOL=$1
python -m paper_2103_07329_b200.build > /dev/null
python scripts/sanitize_cases.py > gpurun_out/san_plain.log 2>&1 || { echo "plain failed"; tail gpurun_out/san_plain.log; exit 1; }
compute-sanitizer --tool $TOOL --print-limit 50 python scripts/sanitize_cases.py > gpurun_out/san_$TOOL.log 2>&1; echo "$TOOL rc=$?"
tail -15 gpurun_out/san_$TOOL.log
