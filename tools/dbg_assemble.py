import sys, torch
import paper_1705_04384_b200 as fd
geom, ne, p = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
params = {0: (), 1: (1.0, 2.0), 2: (0.1,), 3: (1.0, 2.0, 1.0)}[geom]
d = 2 if geom == 1 else 3
ctx = fd.Context(0)
try:
    A = fd.colloc_assemble(ctx, d, p, ne, geom, params)
    print("ok", geom, ne, p, A.nnz)
except Exception as e:
    print("FAIL", geom, ne, p, e)
