# ncu --set full capture of selected C5 kernels (run on the GPU box after a plain run exits 0)
# usage: bash tools/prof_c5.sh TAG "regex" COUNT
TAG=${1:-c5}; RX=${2:-"k_ds_u_div|k_mpm_rhs|k_ds_prep|k_upwind_col|k_kappa_col"}; CNT=${3:-5}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py --config C5 --steps 2 --warmup 3 --skip-e2e --skip-cpu --profile-steps 0 --also "" > gpurun_out/${TAG}_plain.log 2>&1 || { echo plain run failed; tail gpurun_out/${TAG}_plain.log; exit 1; }
ncu --set full --import-source on --clock-control none -k "regex:${RX}" -c ${CNT} -o gpurun_out/${TAG} python bench.py --config C5 --steps 2 --warmup 3 --skip-e2e --skip-cpu --profile-steps 0 --also "" > gpurun_out/${TAG}_ncu.log 2>&1
echo rc=$?
