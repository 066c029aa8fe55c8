cd $GRAFT_REPO_ROOT
python -X faulthandler -c "
import torch, numpy as np
import paper_2508_12627_b200 as us
print('imported', flush=True)
torch.cuda.set_device(0)
A=np.random.default_rng(0).normal(size=(64,64))
print(us.u_statistic_tensors([A,A],[[0,1],[1,2]],3), flush=True)
d=torch.from_numpy(A).cuda()
print(us.u_statistic_tensors([d,d],[[0,1],[1,2]],3), flush=True)
print(us.profile(True, True, 0), flush=True)
print(us.u_statistic_tensors([d,d],[[0,1],[1,2]],3), flush=True)
print(us.profile(False, True, 0), flush=True)
" 2>&1 | head -40
python -X faulthandler bench.py --config C1 --no-cpu-baseline --no-e2e --steps 1 --warmup 1 2>&1 | head -40
