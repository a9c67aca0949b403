import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, '..')
import paper_2603_08982_b200 as P
torch.manual_seed(0)
def rel(a,b): return float((a.double()-b.double()).norm()/b.double().norm())
for d in (64,128):
    for (nq,nk,cq,ck) in ((150,190,4,6),(700,900,5,20)):
        q,k,v=(torch.randn(n,d,device='cuda').bfloat16() for n in (nq,nk,nk))
        prep=P.prepare(q,k,v,cq,ck,seed=0,max_iters=5)
        sizes=prep.q_model.sizes.long().unsqueeze(1)*prep.k_model.sizes.long().unsqueeze(0)
        for name,sel in (('full',torch.ones(cq,ck,dtype=torch.bool)),('empty',torch.zeros(cq,ck,dtype=torch.bool)),('half',torch.rand(cq,ck)<0.5)):
            mask=P.mask_from_selected(sel.cuda(),sizes)
            a=P.sparse_attend(prep.q,prep.k,prep.v,prep.q_model,prep.k_model,mask,dtype=torch.float32)
            b=P.sparse_attend(prep.q,prep.k,prep.v,prep.q_model,prep.k_model,mask,dtype=torch.bfloat16)
            torch.cuda.synchronize()
            print(f"d={d} nq={nq} nk={nk} {name}: rel-L2 bf16 vs fp32 = {rel(b.output,a.output):.3e}  lse maxdiff={float((a.lse-b.lse).abs().max()):.3e} finite={bool(torch.isfinite(b.output.float()).all())}", flush=True)
