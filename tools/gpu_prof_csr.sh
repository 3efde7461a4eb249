cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
tools/exp_red_peak.bin > gpurun_out/red_peak.txt 2>&1
ARGS="--steps 1 --csr 10000000,10000,100000000,200,20"
python tools/prof_step.py $ARGS > gpurun_out/plain_c3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/prof_step.py $ARGS > gpurun_out/ncu_l_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:cs_csr_stream -s 0 -c 1 -o gpurun_out/full_cs_csr_stream python tools/prof_step.py $ARGS > gpurun_out/ncu_full_c3.log 2>&1
echo "rc $?"
cat gpurun_out/red_peak.txt
