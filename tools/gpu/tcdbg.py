import sys, numpy as np, torch
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import test_gpu_tc as t
from configs import config2
p, ctx = t.env("c2s")
nq, N = 24, ctx.n
for (blocks,n1,n2,T) in [(1,32,8,1),(3,32,32,1),(1,32,32,2)]:
    ctw=2*nq*N; rows=blocks*n2
    diags=t.uniform(ctx,nq,rows*n1,5).view(blocks,n2*n1,nq,N)
    ptrs=[diags[r//n2,(r%n2)*n1+k].data_ptr() for r in range(rows) for k in range(n1)]
    packed=ctx.bsgs_tc_pack(ptrs,rows,n1,nq)
    baby=t.uniform(ctx,nq,T*n1*2,6).view(T,n1,2,nq,N)
    inner=torch.full((n2,T,blocks,2,nq,N),-1,dtype=torch.int64,device="cuda")
    ctx.bsgs_mac_tc(inner,T*blocks*ctw,ctw,blocks*ctw,baby,n1*ctw,packed,blocks,n2,n1,nq,tokens=T)
    ref=torch.empty_like(inner)
    for b in range(blocks):
        ctx.bsgs_mac_tokens(ref[:,:,b],T*blocks*ctw,blocks*ctw,baby,n1*ctw,diags[b],nq,n1,n2,nq,tokens=T)
    g=t.host(inner); r=t.host(ref)
    bad=(g!=r)
    print("case",blocks,n1,n2,T,"bad frac",bad.mean(), "unwritten", (g==np.uint64(2**64-1)).mean())
    idx=np.argwhere(bad)
    if len(idx):
        print(" bad limbs", np.unique(idx[:,4])[:30])
        print(" bad t sample", np.unique(idx[:,5]%8), "count by t mod 4", np.bincount(idx[:,5]%4))
        print(" bad j", np.unique(idx[:,0])[:40], "blocks", np.unique(idx[:,2]), "c", np.unique(idx[:,3]))
        for e in idx[:5]:
            e=tuple(e); q=p["chain"][e[4]]
            print("  ",e, int(g[e]), int(r[e]), q, (int(g[e])-int(r[e]))%q)
    # check packed A bytes for one coefficient: limb 1, t 0
    pk=packed.cpu().numpy()
    KC=(5*n1+31)//32*2; RG=(rows+7)//8; KB=KC*128
    li=0  # tc limb 0 = chain limb 1
    tt=3
    base=(li*N+tt)*RG*KB
    ok=True
    dh=t.host(diags)
    for rr in range(rows):
        for k in range(n1):
            w=int(dh[rr//n2,(rr%n2)*n1+k,1,tt])
            for a in range(5):
                kp=a*n1+k
                off=base+(rr//8)*KB+(kp//16)*128+(rr%8)*16+kp%16
                if pk[off]!=(w>>(8*a))&255: ok=False
    print(" packed A ok", ok)
