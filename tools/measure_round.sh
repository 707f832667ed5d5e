# Round-end measurement set (run on the GPU box from the repo root):
# bench lines for C1-C5 and the reference arm, the C2 ncu launch list and one
# ncu --set full capture of the C2 step's top kernels.
set -x
python bench.py > gpurun_out/b_C2.log 2> gpurun_out/b_C2.err
python bench.py --config C1 --steps 100 > gpurun_out/b_C1.log 2> gpurun_out/b_C1.err
python bench.py --config C3 --steps 100 > gpurun_out/b_C3.log 2> gpurun_out/b_C3.err
python bench.py --config C4 > gpurun_out/b_C4.log 2> gpurun_out/b_C4.err
python bench.py --config C5 --steps 60 --skip-cpu > gpurun_out/b_C5.log 2> gpurun_out/b_C5.err
python bench.py --impl reference > gpurun_out/b_ref_C2.log 2> gpurun_out/b_ref_C2.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv python bench.py --steps 40 --warmup 3 --skip-e2e --skip-cpu --profile-steps 0 > gpurun_out/ncu_ll.log 2>&1
ncu --set full --import-source on --clock-control none -k "regex:k_ds_sweep|k_part_solve|k_factor1_t|k_gj_pp|k_upwind|k_kappa|k_gemv|k_ds_u_div|k_mpm_rhs" -c 18 -o gpurun_out/full_c2_v5 python bench.py --steps 6 --warmup 3 --skip-e2e --skip-cpu --profile-steps 0 > gpurun_out/ncu_full.log 2>&1
echo done
