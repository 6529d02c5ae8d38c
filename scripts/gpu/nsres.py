import sys, numpy as np
sys.path.insert(0, '.')
import bench
import paper_1311_1695_b200 as L
a = L.build_laplacian(L.config_graph("C1"))
pairs, rep = L.dacg_smallest(a, 3, delta=1e-10)
U = pairs.vectors
print(type(U), U.shape, U.dtype, U.flags['C_CONTIGUOUS'], float(np.abs(U).max()))
y = L.spmv(a, U[:, 0])
print('spmv', float(np.abs(y).max()), float(np.linalg.norm(y - pairs.values[0] * U[:, 0])))
y2 = L.spmv(a, np.ascontiguousarray(U[:, 0]))
print('spmv contig', float(np.linalg.norm(y2 - pairs.values[0] * U[:, 0])))
print(bench.north_star_residual(a, pairs))
