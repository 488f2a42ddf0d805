cd $GRAFT_REPO_ROOT
for C in 3 4 5; do CX_SEL_TRACE=1 CX_PKG_ROOT=.variants/exp timeout 120 python -c "
import torch,sys
sys.path.insert(0,'.variants/exp')
from paper_2601_01298_b200 import device as cxd
torch.cuda.set_device(0)
g=torch.Generator(device='cuda').manual_seed(0)
G=48; keys=torch.randn(G,8192,64,device='cuda',generator=g); q=torch.randn(G,7,64,device='cuda',generator=g)
a=cxd.attention_grouped(keys,q)
cxd.set_option('select_impl','tc'); cxd.set_option('select_cluster',$C)
cxd.select_grouped(keys,a,164,0.5); torch.cuda.synchronize()
"; done
