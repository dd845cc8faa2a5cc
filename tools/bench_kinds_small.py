import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_09790_b200 as cs
p = cs.DeviceProblem.generate("poisson27", 32, 32, 32).set_precond("jacobi")
for k in sys.argv[1:]:
    print(k, p.bench_spmv(k, 2), flush=True)
