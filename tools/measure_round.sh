# Round-end measurement set (run on the GPU box from the repo root):
# the default bench line (C5 headline + C2), C1/C3/C4 lines, the reference
# arm, the C5 ncu launch list, and one ncu --set full capture of the C5
# step's top kernels. Each ncu pass runs only after its plain command exited 0.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py > gpurun_out/b_default.log 2> gpurun_out/b_default.err || exit 1
python bench.py --config C1 --steps 100 --also "" > gpurun_out/b_C1.log 2> gpurun_out/b_C1.err
python bench.py --config C3 --steps 100 --also "" > gpurun_out/b_C3.log 2> gpurun_out/b_C3.err
python bench.py --config C4 --also "" > gpurun_out/b_C4.log 2> gpurun_out/b_C4.err
python bench.py --impl reference > gpurun_out/b_ref.log 2> gpurun_out/b_ref.err
python bench.py --steps 10 --warmup 3 --skip-e2e --skip-cpu --profile-steps 0 --also "" > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C5.csv python bench.py --steps 10 --warmup 3 --skip-e2e --skip-cpu --profile-steps 0 --also "" > gpurun_out/ncu_ll.log 2>&1
ncu --set full --import-source on --clock-control none -k "regex:k_ds_blk_factor|k_ds_blk_solve|k_part_solve|k_cr_gemv|k_mpm_rhs_w|k_mpm_edges|k_ds_u_div|k_ds_prep|k_upwind_col|k_kappa_col" -c 12 -o gpurun_out/full_c5_r02 python bench.py --steps 3 --warmup 3 --skip-e2e --skip-cpu --profile-steps 0 --also "" > gpurun_out/ncu_full.log 2>&1
echo done
