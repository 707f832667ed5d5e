python -m pytest tests/test_gpu_spaces.py -k "not C5" -x -q -p no:cacheprovider -s > gpurun_out/spaces.log 2>&1; echo spaces rc=$?
python -m pytest tests/test_gpu_full_runs.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/full.log 2>&1; echo full rc=$?
python bench.py --steps 80 --warmup 3 --skip-e2e --skip-cpu --also "" > gpurun_out/b_hg8.log 2>&1; echo b8 rc=$?
MPM2P_HOM_GROUP=1 python bench.py --steps 80 --warmup 3 --skip-e2e --skip-cpu --also "" > gpurun_out/b_hg1.log 2>&1; echo b1 rc=$?
