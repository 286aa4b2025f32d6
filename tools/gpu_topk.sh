cd $GRAFT_REPO_ROOT
export APPD_DEBUG_ROUNDS=1
python - > gpurun_out/topk.log 2>&1 <<'PY'
import torch, numpy as np, sys
sys.path.insert(0, '.')
import paper_2407_07058_b200 as P
from synth import generators as G
X = torch.from_numpy(np.ascontiguousarray(G.config("C4"), np.float32)).cuda()
for topk in [8, 16]:
    c = P.Context(timing=True, topk=topk, finish_k=0)
    for _ in range(2):
        M = c.solve_points(X); torch.cuda.synchronize()
    st = c.stats()
    print("topk", topk, {k: st[k] for k in ["rounds","ms_mst","ms_total","ms_tcscan","rescan_rows","rescan_blocks"]}, flush=True)
    c.close(); del M
PY
echo "exit $?"; grep -v "round [1-9]" gpurun_out/topk.log | tail -30
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -5 gpurun_out/pytest_gpu.log
bash tools/prof_launch.sh
