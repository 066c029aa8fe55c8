# quick GPU shake-out: build check, tiny parity, then the GPU test suite
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "
import numpy as np, paper_2508_12627_b200 as us
print(us.device_count())
x=np.array([[1.],[2.],[3.]]); print('prod2', us.u_statistic('prod2', x), us.v_statistic('prod2', x))
rng=np.random.default_rng(0); A=rng.normal(size=(150,150)); B=rng.normal(size=(150,150))
print('gemm err', np.abs(us.einsum([A,B],[[0,1],[1,2]],[0,2]) - A@B).max())
"
timeout 900 python -m pytest tests -m gpu -q -v 2>&1 | grep -v "^  File" | tail -80
