import sys, os, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from gpu_helpers import *
topo, data = make_case(16, dim=2, p=0.3, mode='local', seed=16, B=3)
g = graph_for(topo)
st = D.dnls_graph_stats(g); print(st, flush=True)
H = []
for b in range(3):
    prob = oracle_problem(topo, data, b)
    _, Hb, _ = prob.linearize(olie.to_homog(data['poses0'][b])); H.append(Hb)
H = np.stack(H); n = H.shape[1]
ws = D.alloc_workspace(g, 3)
D.dnls_import_matrix(g, 3, torch.from_numpy(H).to(DEV), ws); torch.cuda.synchronize(); print('import ok', flush=True)
s = torch.full((3,), -1, dtype=torch.int32, device=DEV)
D.dnls_factorize(g, 3, ws, s); torch.cuda.synchronize(); print('factor ok', s.tolist(), flush=True)
x = torch.zeros(3, n, dtype=torch.float64, device=DEV)
D.dnls_solve_factored(g, 3, ws, torch.ones(3, n, dtype=torch.float64, device=DEV), x); torch.cuda.synchronize(); print('solve ok', flush=True)
