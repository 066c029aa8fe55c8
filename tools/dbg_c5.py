import sys; sys.path.insert(0,'.')
import numpy as np, paper_2508_12627_b200 as us
from paper_2508_12627_b200.workloads import generate
f, sig, m, _ = generate("C5", 1024)
txt, tot = us.plan_summary(sig, m, 1024, us.Config(memory_cap_entries=2**40), inputs_symmetric=True)
print(txt)
try:
    r = us.u_terms(f, sig, m, us.Config(memory_cap_entries=2**40))
    print("ok", r.value)
except Exception as e:
    print("ERR", e)
