# per-phase cycles of select_tc (experiments build: tools/build_variant.sh exp WORKTREE -DCX_EXPERIMENTS)
# usage on the box: bash tools/_seltrace.sh "EXCHANGE C" ...   (exchange 1 = cluster, 2 = cooperative)
cd $GRAFT_REPO_ROOT
for cfg in "$@"; do set -- $cfg; CX_SEL_TRACE=1 CX_PKG_ROOT=.variants/exp timeout 120 python -c "
import torch,sys
sys.path.insert(0,'.variants/exp')
from paper_2601_01298_b200 import device as cxd
torch.cuda.set_device(0)
g=torch.Generator(device='cuda').manual_seed(0)
G=48; keys=torch.randn(G,8192,64,device='cuda',generator=g); q=torch.randn(G,7,64,device='cuda',generator=g)
a=cxd.attention_grouped(keys,q)
cxd.set_option('select_impl','tc'); cxd.set_option('select_exchange',$1); cxd.set_option('select_cluster',$2)
cxd.select_grouped(keys,a,164,0.5); torch.cuda.synchronize()
e0,e1=torch.cuda.Event(True),torch.cuda.Event(True); e0.record(); cxd.select_grouped(keys,a,164,0.5); e1.record(); torch.cuda.synchronize(); print('exchange',$1,'C',$2,'ms',e0.elapsed_time(e1))
"; done
