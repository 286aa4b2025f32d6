import sys, ctypes
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2407_07058_b200 as P
from synth import generators as G
L = P.load()
L.appd_debug_tc_gram.argtypes = [ctypes.c_void_p]*2 + [ctypes.c_int64]*2 + [ctypes.c_void_p]*2
ctx = P.Context()
for (n, d, kind) in [(256, 2, 'uniform'), (512, 64, 'blobs'), (300, 16, 'dups')]:
    X = torch.from_numpy(G.random_points(n, d, 1, kind)).cuda()
    npad = (n + 511)//512*512
    tc = torch.zeros((512, npad), device='cuda'); ref = torch.zeros((512, npad), device='cuda')
    s = L.appd_debug_tc_gram(ctx._h, X.data_ptr(), n, d, tc.data_ptr(), ref.data_ptr())
    a = tc.cpu().numpy(); b = ref.cpu().numpy()
    print(n, d, kind, 'status', s, 'maxabs', np.abs(a-b).max(), 'ref range', b.min(), b.max())
    print(' tc[0,:6]', a[0,:6]); print(' ref[0,:6]', b[0,:6])
    print(' tc[1,:6]', a[1,:6]); print(' ref[1,:6]', b[1,:6])
    print(' tc[9,:6]', a[9,:6]); print(' ref[9,:6]', b[9,:6])
    bad = np.argwhere(np.abs(a-b) > 1e-2 * (1 + np.abs(b)))
    print(' nbad', len(bad), bad[:5])
