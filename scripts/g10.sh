mkdir -p gpurun_out
( for c in "C4p 1" "C4p 4" "C4b 1" "C4b 8" "C3 32"; do set -- $c; python scripts/sc_time.py $1 $2 2>&1 | tail -1; done ) > gpurun_out/sc_tab.log 2>&1
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
