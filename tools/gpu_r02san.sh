# compute-sanitizer memcheck over every kernel family at small sizes (tools/sanitize_run.py); output kept as-is
O=gpurun_out/r02san; mkdir -p $O
which compute-sanitizer > $O/memcheck.log 2>&1
timeout 1200 compute-sanitizer --tool memcheck --leak-check no python tools/sanitize_run.py >> $O/memcheck.log 2>&1; echo "memcheck rc=$?" >> $O/memcheck.log
tail -5 $O/memcheck.log
