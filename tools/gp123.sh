# SYRK SM-reserve sweep after the POTRF/TRSM speedups (big,small,m_threshold)
for r in 8,24,8192 6,24,8192 6,16,8192 4,24,8192 8,16,8192 6,20,8192 5,24,8192; do
  echo "== $r"; STAN_CL_SYRK_RESERVE=$r python tools/quick_time.py 8192 16384 | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['n'], round(d['fwd_ms'], 3))"
done
