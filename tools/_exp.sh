timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "TestExecutor and not large" 2>&1 | tail -4
compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -q -x -k "TestExecutor or executor_random_masks" 2>&1 | tail -4
