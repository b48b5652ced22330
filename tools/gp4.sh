python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for cfg in mid,mid,big big,big,big mid,mid,mid big,mid,big; do
  echo "cfg=$cfg"; STAN_CL_GEMM_CFG=$cfg python tools/quick_time.py 16384 2>&1 | tail -1
done
python - <<'PY'
import sys, torch; sys.path.insert(0,'.')
import paper_1907_01063_b200 as sc
from paper_1907_01063_b200 import inputs
n=16384
x=torch.from_numpy(inputs.gp_x(n)).cuda(); K=sc.gp_exp_quad_cov(x,1,1,1e-6); W=torch.from_numpy(inputs.lbar(n)).cuda()
L=torch.empty_like(K); A=torch.empty_like(K)
sc.cholesky(K,out=L); sc.cholesky_adjoint(L,W,out=A); torch.cuda.synchronize()
sc.profile_reset(); sc.profile_enable(True)
sc.cholesky(K,out=L); sc.cholesky_adjoint(L,W,out=A); torch.cuda.synchronize()
sc.profile_enable(False)
import json
for k,v in sc.profile_read().items(): print(k, json.dumps(v))
PY
ncu --set full --clock-control none --import-source on -k regex:gemm_dmma -s 30 -c 4 -o gpurun_out/prof_gemm_r01 python tools/quick_time.py 8192 > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"potrf|trsm" -s 20 -c 2 -o gpurun_out/prof_panel_r01 python tools/quick_time.py 4096 > gpurun_out/ncu_full2.log 2>&1
tail -3 gpurun_out/ncu_full.log
