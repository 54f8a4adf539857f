mkdir -p gpurun_out
python -m pytest tests/test_parity_shapes_gpu.py -m gpu -x -q -k "u8_line" > gpurun_out/pytest_u8.log 2>&1; tail -5 gpurun_out/pytest_u8.log
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
