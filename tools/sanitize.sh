#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_run.py -> gpurun_out/sanitizer_*.txt
mkdir -p gpurun_out
python tools/sanitize_run.py all > gpurun_out/sanitizer_plain.txt 2>&1; tail -1 gpurun_out/sanitizer_plain.txt
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 python tools/sanitize_run.py all > gpurun_out/sanitizer_memcheck.txt 2>&1; tail -2 gpurun_out/sanitizer_memcheck.txt
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python tools/sanitize_run.py all > gpurun_out/sanitizer_racecheck.txt 2>&1; tail -2 gpurun_out/sanitizer_racecheck.txt
timeout 1500 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_run.py all > gpurun_out/sanitizer_synccheck.txt 2>&1; tail -2 gpurun_out/sanitizer_synccheck.txt
# canary: the same tools must flag a known out-of-bounds store and a shared-memory race
compute-sanitizer --tool memcheck ./tools/sanitizer_canary.bin > gpurun_out/sanitizer_canary_memcheck.txt 2>&1; grep -c "Invalid __global__ write" gpurun_out/sanitizer_canary_memcheck.txt
compute-sanitizer --tool racecheck ./tools/sanitizer_canary.bin > gpurun_out/sanitizer_canary_racecheck.txt 2>&1; tail -1 gpurun_out/sanitizer_canary_racecheck.txt
