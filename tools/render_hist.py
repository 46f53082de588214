import sys, numpy as np
sys.path.insert(0,'.')
import paper_2506_19139_b200 as sof
from paper_2506_19139_b200.workloads import CONFIGS, orbit_cameras, synthetic_scene
cfg=CONFIGS["C2"]
scene=synthetic_scene(cfg["gaussians"],2)
cams=orbit_cameras(cfg["views"],cfg["width"],cfg["height"]).subset(np.array([0,1,2]))
ctx=sof.Context(0); views=sof.ViewSet.build(scene,cams,ctx=ctx)
for v in range(3):
    r=sof.render_view(views,v,sof.DEPTH_EXACT,counts=True)
    c=r["counts"].ravel()
    edges=[0,1,2,33,65,129,257,513,1025,4097,10**9]
    h=np.histogram(c,bins=edges)[0]
    print(v, "mean",c.mean(),"max",c.max(), "total",c.sum())
    for a,b,k in zip(edges[:-1],edges[1:],h): print(f"   [{a},{b}) {k} px  {c[(c>=a)&(c<b)].sum()/c.sum()*100:.1f}% of entries")
