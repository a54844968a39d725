import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch, paper_2410_10989_b200 as lk
from paper_2410_10989_b200.fused_linear_cross_entropy import fused_linear_cross_entropy_forward as f
torch.manual_seed(0)
bt,h,v=8192,4096,128256
x=(torch.rand(bt,h,device="cuda")*2-1).bfloat16(); w=((torch.rand(v,h,device="cuda")*2-1)/64).bfloat16()
t=torch.randint(0,v,(bt,),device="cuda"); t[::10]=-100
ref=None; bad=0
for i in range(6):
    loss,_,_,_,gx,gw,_=f(x,w,t,compute_grad_input=True,compute_grad_weight=True)
    cur=(loss.item(),gx.clone(),gw.clone())
    if ref is None: ref=cur
    else:
        ok = cur[0]==ref[0] and torch.equal(cur[1],ref[1]) and torch.equal(cur[2],ref[2])
        bad += not ok
        print(i, ok, (cur[1].float()-ref[1].float()).abs().max().item(), (cur[2].float()-ref[2].float()).abs().max().item())
z=(torch.randn(8192,v,device="cuda")*3).bfloat16()
outs=[]
for i in range(4):
    zz=z.clone().requires_grad_(True); l=lk.LigerCrossEntropyLoss()(zz,t); l.backward(); outs.append((l.item(), zz.grad.clone()))
print("ce", all(o[0]==outs[0][0] and torch.equal(o[1],outs[0][1]) for o in outs))
print("flce bad", bad)
