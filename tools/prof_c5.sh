# ncu --set full captures of the C5 step's kernels (run on the GPU box from the
# repo root, after a plain run exits 0). The MPM-2P kernels in one pass; the
# interface GEMV separately, skipping the initial solve's rcond-estimate launches.
TAG=${1:-full_c5}
set -x
python bench.py --config C5 --steps 2 --warmup 3 --skip-e2e --skip-cpu --profile-steps 0 --also "" > gpurun_out/${TAG}_plain.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none \
    -k "regex:k_ds_blk_factor|k_ds_blk_solve|k_part_solve|k_mpm_rhs_w|k_mpm_edges|k_ds_u_div|k_ds_prep|k_upwind_col|k_kappa_col|k_recon_mpm" \
    -c 11 -o gpurun_out/${TAG}_a python bench.py --config C5 --steps 2 --warmup 3 --skip-e2e --skip-cpu --profile-steps 0 --also "" > gpurun_out/${TAG}_a.log 2>&1
ncu --set full --import-source on --clock-control none -k "regex:k_cr_gemv" --launch-skip 300 -c 15 \
    -o gpurun_out/${TAG}_b python bench.py --config C5 --steps 2 --warmup 3 --skip-e2e --skip-cpu --profile-steps 0 --also "" > gpurun_out/${TAG}_b.log 2>&1
echo rc=$?
