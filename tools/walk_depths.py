import numpy as np, gen, paper_1702_03657_b200 as pf
from tests import image_walker as iw
import collections
for cid in [3]:
    ps=gen.patterns(cid); h=iw.parse(pf.Trie(ps).image())
    t=gen.text(cid,0,300000).tobytes()
    node,label=h['node'],h['label']
    depths=collections.Counter(); tails=0; single=0; multi=0
    for i in range(len(t)-4):
        key=int.from_bytes(t[i:i+4],'little')
        if not iw.filter_pass(h,key,i): continue
        v=int(h['root'][t[i]])
        if v==0: continue
        d=1; j=i+1
        while j<len(t):
            if node[v]&iw.TAIL: tails+=1; break
            s_,e_=int(node[v])&iw.MASK,int(node[v+1])&iw.MASK
            if s_==e_: break
            if e_-s_==1: single+=1
            else: multi+=1
            labs=label[s_:e_]; k=np.searchsorted(labs,t[j])
            if k>=len(labs) or labs[k]!=t[j]: break
            v=s_+int(k)+1; d+=1; j+=1
        depths[d]+=1
    tot=sum(depths.values())
    print('walks',tot,'per byte',tot/len(t),'tails',tails,'single-child steps',single,'multi',multi)
    for d in sorted(depths): print(d, depths[d], round(depths[d]/tot,4))
