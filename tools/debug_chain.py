"""GPU debug helper: C2-like chain, layer by layer, host vs device inputs."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as ora, paper_1801_10585_b200 as spc
from synth import *
x = mnist_like(16, SEED_BASE + 1, values="dyadic")
chans=[1,8,16,32]; ks=[117,29,7]
ws=[sparse_filter(1,8,(3,3),1.0,80,values="dyadic",scale=0.25), sparse_filter(8,16,(3,3),1.0,81,values="dyadic4",scale=0.125), sparse_filter(16,32,(3,3),1.0,82,values="dyadic4",scale=0.125)]
bs=[bias_vector(chans[i+1],90+i,values="dyadic") for i in range(3)]
cur=x
for i in range(2):
    yk,yv,_,_=ora.conv_fwd(cur,ws[i],bs[i],attn=1,k=ks[i]); cur=COO(cur.batch,chans[i+1],cur.dims,yk,yv)
    rk,rv,_=ora.relu(cur); cur=COO(cur.batch,chans[i+1],cur.dims,rk,rv)
    pk,pv,_=ora.maxpool(cur,(2,2)); cur=COO(cur.batch,chans[i+1],tuple(-(-d//2) for d in cur.dims),pk,pv)
W = spc.SparseFilter.from_arrays(ws[2].keys, ws[2].values, 16, 32, (3,3))
mode = sys.argv[1] if len(sys.argv) > 1 else "host"
if mode == "host":
    X = spc.SparseMap.from_arrays(cur.keys, cur.values, cur.batch, cur.channels, cur.dims)
else:
    X0 = spc.SparseMap.from_arrays(cur.keys, cur.values, cur.batch, cur.channels, cur.dims)
    pad = 7424 - cur.nnz
    keys = torch.cat([X0.keys, torch.full((pad,), 123456789123, dtype=torch.int64, device="cuda")])
    vals = torch.cat([X0.values, torch.ones(pad, device="cuda")])
    X = spc.SparseMap(keys, vals, cur.batch, cur.channels, cur.dims, 7424, torch.tensor([cur.nnz], device="cuda"))
Y = spc.sparse_conv_fwd(X, W, torch.from_numpy(bs[2]).cuda(), "magnitude", ks[2])
yk, yv = Y.trimmed()
ok, ov, _, _ = ora.conv_fwd(cur, ws[2], bs[2], attn=1, k=ks[2])
print(mode, "nnz", yk.shape[0], ok.shape[0], "keys equal", np.array_equal(yk.cpu().numpy().view(np.uint64), ok))
