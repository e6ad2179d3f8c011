cd $GRAFT_REPO_ROOT
TAG=${1:-r2k}
NKS_BUILD_TAG=abl NKS_BUILD_DEFS=-DNKS_R2_ABLATE python -m paper_2209_08001_b200.build > gpurun_out/${TAG}_abl_build.log 2>&1
NKS_LIB=$PWD/paper_2209_08001_b200/lib/libnks_abl.so NKS_RAS2D_PROF=1 timeout 600 python -c "
import sys; sys.path.insert(0,'.')
import torch, numpy as np, nks_inputs as ni
from paper_2209_08001_b200 import Solver
shape=(512,512)
c,eta=ni.initial_fields(shape,0)
g=Solver(shape, ni.model_default(), ni.solver_default(), nsub=(4,4), overlap=2)
g.set_fields(c,eta,None)
X=g.get_state(); g.pc_setup(X,0.5)
r=torch.rand((4,)+shape,dtype=torch.float64,device='cuda')
for _ in range(30): g.pc_apply(r)
torch.cuda.synchronize()
" > gpurun_out/${TAG}_r2prof.log 2>&1
for dbg in 0 4 16 32 64 256 260; do
  NKS_LIB=$PWD/paper_2209_08001_b200/lib/libnks_abl.so NKS_RAS2D_DBG=$dbg timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import torch, numpy as np, nks_inputs as ni
from paper_2209_08001_b200 import Solver
shape=(512,512)
c,eta=ni.initial_fields(shape,0)
g=Solver(shape, ni.model_default(), ni.solver_default(), nsub=(4,4), overlap=2)
g.set_fields(c,eta,None)
X=g.get_state(); g.pc_setup(X,0.5)
r=torch.rand((4,)+shape,dtype=torch.float64,device='cuda')
for _ in range(5): g.pc_apply(r)
torch.cuda.synchronize()
g.set_profiling(True); g.phase_times(reset=True)
for _ in range(20): g.pc_apply(r)
ph=g.phase_times(reset=True)
print('dbg $dbg apply ms', ph['ras_apply']['ms']/ph['ras_apply']['count'])
" >> gpurun_out/${TAG}_r2dbg.log 2>&1
done
