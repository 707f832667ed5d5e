# Round check on the GPU box (from the repo root): the GPU suite, smoke, the
# default bench line, then the C5 ncu launch list and full captures (each ncu
# pass only after its plain command exited 0).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
python bench.py > gpurun_out/b_default.log 2> gpurun_out/b_default.err; echo bench rc=$?
if [ "$1" = "prof" ]; then
python bench.py --steps 10 --warmup 3 --skip-e2e --skip-cpu --profile-steps 0 --also "" > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C5.csv python bench.py --steps 10 --warmup 3 --skip-e2e --skip-cpu --profile-steps 0 --also "" > gpurun_out/ncu_ll.log 2>&1
bash tools/prof_c5.sh ${2:-full_c5}
fi
