cd $GRAFT_REPO_ROOT
export APPD_DEBUG_ROUNDS=1
python - > gpurun_out/cache_dbg.log 2>&1 <<'PY'
import torch, numpy as np, sys
sys.path.insert(0, '.')
import paper_2407_07058_b200 as P
from synth import generators as G
for name in ["C2", "C4"]:
    X = torch.from_numpy(np.ascontiguousarray(G.config(name), np.float32)).cuda()
    for topk in [16, -1]:
        c = None
        c = P.Context(timing=True, topk=topk, finish_k=(0 if topk > 0 else -1))
        M = c.solve_points(X); torch.cuda.synchronize()
        M2 = c.solve_points(X); torch.cuda.synchronize()
        st = c.stats()
        print(name, "topk", topk, {k: st[k] for k in ["rounds","ms_mst","ms_dendrogram","ms_fill","ms_total","ms_tcscan","topk","rescan_rounds","rescan_rows","rescan_blocks","cache_invalid_rows","tc_fallback_rows","cm_k"]}, flush=True)
        if topk == 16: Mc = M.clone()
        else: print("equal to no-cache:", bool(torch.equal(Mc.view(torch.int32), M.view(torch.int32))), flush=True)
        c.close()
        del M, M2
PY
echo "dbg exit $?"; tail -40 gpurun_out/cache_dbg.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -30 gpurun_out/pytest_gpu.log
