mkdir -p gpurun_out
( for c in "T1_64_1 64" "T1_64_2 64" "T1_128_1 64" "T1_128_2 64" "C4p 1" "C4p 4" "C2 100" "C3 32" "C4a 1"; do set -- $c; python scripts/quick_time.py $1 $2 2>&1 | grep -E "beamform [0-9]|rror"; done ) > gpurun_out/q13.log 2>&1
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu13.log 2>&1; tail -3 gpurun_out/pytest_gpu13.log
