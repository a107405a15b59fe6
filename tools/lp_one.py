import sys; sys.path.insert(0, ".")
import paper_2301_08695_b200 as bx
from paper_2301_08695_b200 import workloads as W
gen, n, algos, kw, f = W.CONFIGS[sys.argv[1]]
meta, _ = bx.build_grouped(gen(), **kw)
sol = bx.solve_relaxed(meta, bx.CommModel(*W.COMM_TEST))
print(sol.iterations, sol.solver)
