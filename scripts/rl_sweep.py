import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/scripts')
import paper_1804_06087_b200 as rk
from bench import lat_profile, TAU_NS
from paper_1804_06087_b200.scheduler import ActorCritic
K,B=3,[16,32,48,64]
ctx=rk.Context(0); ctx.load_ensemble(K,10)
N=2_000_000
acc=np.array([0.80,0.78,0.83,0.75,0.82,0.81,0.84])
for ref in (128.0, 572.0):
    arr=torch.empty(N,dtype=torch.int64,device='cuda'); ctx.sine_arrivals(arr,N,ref,500*TAU_NS,50_000_000,0.1,7)
    cfg=rk.RewardCfg(B=B,beta=1.0,tau_ns=TAU_NS,lat_ns=lat_profile(K,B),arrival_ns=arr)
    for lp,lv in ((0.05,0.005),(0.2,0.01),(0.5,0.01),(1.0,0.02)):
        ag=ActorCritic(ctx,cfg,acc,arr,L=16,H=64,n_steps=32,seed=0)
        try:
            c=ag.train(60,E=512,lr_pi=lp,lr_v=lv)
            print(ref,lp,lv,[round(x['reward_per_request'],3) for x in c[::10]], round(c[-1]['overdue_frac'],3), round(c[-1]['mean_models'],2), round(c[-1]['loss_v'],3), flush=True)
        except Exception as e:
            print(ref,lp,lv,'ERR',e, flush=True)
