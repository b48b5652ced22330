# launch list of one forward at n=4096 (critical-path study)
export STAN_CL_GRAPH=0
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fwd4096_launches.csv python tools/fwd_once.py 4096 > /dev/null 2>&1
wc -l gpurun_out/fwd4096_launches.csv
