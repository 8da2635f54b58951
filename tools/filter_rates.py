import numpy as np, gen, paper_1702_03657_b200 as pf
from tests import image_walker as iw
for cid in [2,3,4,5]:
    ps=gen.patterns(cid); h=iw.parse(pf.Trie(ps).image())
    t=gen.text(cid,0,200000).tobytes()
    n=len(t)-4; surv=0; keep=0; per_lane=[]
    for i in range(0,n):
        key=int.from_bytes(t[i:i+4],'little')
        if iw.filter_pass(h,key,i):
            surv+=1
            v=int(h['root'][t[i]])
            if v:
                w=int(h['node'][v])
                k=(w&(iw.TERM|iw.TAIL))!=0
                if not k:
                    c1=t[i+1]; bm=h['level1'][v-1]
                    k=(int(bm[c1>>5])>>(c1&31))&1
                keep+=bool(k)
    print(cid, h['filter_kind'], 'surv %.4f keep %.4f'%(surv/n, keep/n))
