"""2:4 violation survey: for candidate groupings of 4 pixels, how many needle rows (C2 sample,
and a 10-object clutter scene) have a group with 3-4 non-zero D_n.  CPU, uses the oracle."""
import sys, numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__)))))
import synth, oracle
def imgs_c2(n=1024):
    cfg=synth.config_c2(); m=cfg['mesh']; O=cfg['origins']
    sel=np.sort(np.random.default_rng(1).choice(len(O),n,replace=False))
    return oracle.rici_generate(m.vertices, m.indices, O[sel], 0.3, 64)['images'].astype(np.int32)
def imgs_scene(n=512):
    objs=[synth.bumpy_torus(120,60,key=(41,k),minor=0.25+0.02*k,amp=0.08) for k in range(10)]
    sc=synth.clutterbox(objs,key=(41,1000))
    O=sc.origins; sel=np.sort(np.random.default_rng(2).choice(len(O),n,replace=False))
    return oracle.rici_generate(sc.vertices, sc.indices, O[sel], 0.3, 64)['images'].astype(np.int32)
for name,img in [("c2",imgs_c2()),("scene",imgs_scene())]:
    D=np.zeros_like(img); D[:,:,1:]=img[:,:,1:]-img[:,:,:-1]
    nz=(D!=0)
    n=len(nz)
    print(name,"density",nz.mean())
    blk=nz.reshape(n,32,2,64)   # [needle, pair j, row-in-pair, col]
    def ev(groups,label):
        # groups: list of 4-tuples of (rowinpair, col) covering 128 pixels
        cnt=np.zeros((n,32),int)
        viol=np.zeros((n,),int)
        for gidx in groups:
            s=sum(blk[:,:,r,c].astype(int) for r,c in gidx)
            viol+= (s>2).sum(1)
        print(f"  {label:28s} violations/needle {viol.mean():.4f}  needles with any {(viol>0).mean():.4f}")
    ev([[(r,c+4*0+k) for k in range(4)] for r in range(2) for c in range(0,64,4)],"consecutive")
    ev([[(r,c+16*k) for k in range(4)] for r in range(2) for c in range(16)],"stride16")
    ev([[(0,c),(0,c+32),(1,c+16),(1,c+48)] for c in range(16)]+[[(1,c),(1,c+32),(0,c+16),(0,c+48)] for c in range(16)],"2row-stride16")
    ev([[(0,c),(1,c+16),(0,c+32),(1,c+48)] for c in range(16)]+[[(1,c),(0,c+16),(1,c+32),(0,c+48)] for c in range(16)],"2row-alt")
    ev([[(r,c+8*k) for k in range(4)] for r in range(2) for c in list(range(8))+list(range(32,40))],"stride8")
