python tools/bench_gp.py 1024 4096 16384 2>&1 | tee gpurun_out/r01_gp_bench.jsonl
python -c "
import time, sys; sys.path.insert(0,'.')
import oracle
from paper_1907_01063_b200 import inputs
n=1024; x=inputs.gp_x(n); y=inputs.gp_y(x)
t=time.perf_counter(); oracle.gp_lpdf_grad(x,y,1.0,1.0,0.1); dt=time.perf_counter()-t
print('oracle gp_lpdf_grad n=1024 s', dt)
" | tee -a gpurun_out/r01_gp_bench.jsonl
