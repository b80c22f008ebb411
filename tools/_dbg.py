import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from conftest import load_golden, rel_err
from paper_2304_04980_b200 import GpuSchurOperator, GpuNestedJacobiPreconditioner
for name in sys.argv[1:]:
    ga, rec = load_golden(name)
    op = GpuSchurOperator(ga, rec["L"], rec["S"])
    v = rec["vec"]
    print(name, "delta", rel_err(op.apply(v), rec["delta"]), flush=True)
    print(name, "outer", rel_err(op.apply_outer_coupling(v), rec["outer"]), flush=True)
