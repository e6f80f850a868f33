import sys, torch, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2509_07120_b200 as bsa
import torch.nn.functional as F
from test_gpu_qkv import _inputs, _ref_qkv
for (Fr,P,S,H) in [(4,1369,5,16),(3,300,5,4)]:
    lay, x, w, b = _inputs(Fr,P,S,H, seed=Fr*7+P+S+H)
    q,k,v,qp,kp = bsa.qkv_projection(x,w,b,H,lay)
    ref = _ref_qkv(x,w,b,H)
    T=lay.total_tokens
    cub = F.linear(x,w,b).view(T,3,H,64).permute(1,2,0,3)
    absw = (x.double().abs() @ w.double().abs().T).view(T,3,H,64).permute(1,2,0,3)
    for i,(name,got) in enumerate((("q",q),("k",k),("v",v))):
        r=ref[i]; e=(got.double()-r).abs(); ec=(cub[i].double()-r).abs()
        ulp = torch.exp2(torch.floor(torch.log2(r.abs().clamp_min(1e-30)))-7)
        print(name, H, "ours max ulps", (e/ulp).max().item(), ">0.5ulp frac", ((e/ulp)>0.5001).double().mean().item(),
              "| cublas max ulps", (ec/ulp).max().item(), ">0.5ulp frac", ((ec/ulp)>0.5001).double().mean().item())
        idx = torch.argmax(e/ulp)
        print("   worst: ref", r.flatten()[idx].item(), "ours", got.flatten()[idx].item(), "cublas", cub[i].flatten()[idx].item(), "sum|xw|", absw[i].flatten()[idx].item())
