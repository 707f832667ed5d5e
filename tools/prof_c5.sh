set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py --config C5 --steps 2 --warmup 3 --skip-e2e --skip-cpu --profile-steps 0 > gpurun_out/c5_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k "regex:k_ds_solve|k_upwind_col|k_kappa_col|k_part_solve|k_mpm_rhs|k_ds_u_div" -c 6 -o gpurun_out/full_c5_r02a python bench.py --config C5 --steps 2 --warmup 3 --skip-e2e --skip-cpu --profile-steps 0 > gpurun_out/ncu_c5.log 2>&1
echo rc=$?
