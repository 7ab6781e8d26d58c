#!/bin/bash
# compute-sanitizer over the round-2 kernels (certified modes, golden parity),
# then the full GPU suite.
O=gpurun_out/san; mkdir -p $O
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_certified.py tests/test_gpu_parity.py -x -q -m gpu -k "certified or golden or lognormal" > $O/memcheck_r02.log 2>&1; echo "memcheck rc=$?"; tail -4 $O/memcheck_r02.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_certified.py -x -q -m gpu -k "goldens" > $O/racecheck_r02.log 2>&1; echo "racecheck rc=$?"; tail -4 $O/racecheck_r02.log
timeout 1500 python -m pytest tests -q -m gpu --durations=10 > $O/pytest_gpu_full.log 2>&1; echo "pytest rc=$?"; tail -14 $O/pytest_gpu_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -4 $O/smoke.log
