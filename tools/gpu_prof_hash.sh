cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python tools/exp_hash_only.py > gpurun_out/hash_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"raw_draws|fy_count|fy_scatter|fy_final|sign_kernel|lemire_write" -s 6 -c 6 \
    -o gpurun_out/full_hash_parallel python tools/exp_hash_only.py > gpurun_out/ncu_hash.log 2>&1
echo rc $?
tail -3 gpurun_out/ncu_hash.log
