import sys, pathlib; sys.path.insert(0, "/root/repo")
import torch, paper_2410_10989_b200 as lk
bt,v=8192,128256
z=(torch.randn(bt,v,device="cuda")*3).bfloat16(); t=torch.randint(0,v,(bt,),device="cuda")
w=torch.rand(v,device="cuda")+0.5
def run(kw):
    for _ in range(3):
        zz=z.clone().requires_grad_(True); lk.LigerCrossEntropyLoss(**kw)(zz,t).backward()
    ts=[]
    for _ in range(10):
        zz=z.clone().requires_grad_(True); e0=torch.cuda.Event(True); e1=torch.cuda.Event(True)
        e0.record(); lk.LigerCrossEntropyLoss(**kw)(zz,t).backward(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ts.sort(); return ts[len(ts)//2]
for kw in [dict(), dict(label_smoothing=0.1), dict(weight=w), dict(weight=w,label_smoothing=0.1)]:
    print(list(kw.keys()), round(run(kw),3), "ms")
