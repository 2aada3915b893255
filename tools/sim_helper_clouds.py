# Simulation (oracle only): would dense clouds of helper chains seeded ahead of a long
# extension shorten the seam tail?  See profiles/r01/sweeps.md.
import sys; sys.path.insert(0,'/root/repo')
import numpy as np, synth, oracle
n=1<<30
b=synth.fill_host('markov',2,0,n)
p=oracle.table1(4,1)
true=oracle.chunk(b,p)
ts=set(true.tolist())
G=335872
def chain(start,k):
    out=[]; c=start
    for _ in range(k):
        if c>=n: break
        c=oracle.next_cut(b,c,p); out.append(c)
    return out
long=[]
for s in range(1, n//G):
    lo=s*G; c=lo; k=0
    while c not in ts and c<n:
        c=oracle.next_cut(b,c,p); k+=1
    if k>30: long.append((k,lo))
print('seams with D>30:', len(long), 'max D', max(long)[0])
CH=2500  # bytes per chunk (approx)
for clouds, members, spacing, step_k in [(6,16,150,10),(10,16,150,10),(10,32,150,8),(12,8,300,8)]:
    out=[]
    for D,lo in long:
        i0=np.searchsorted(true, lo); A=true[i0:i0+160].tolist()
        Bl=chain(lo,260); Bset={c:i for i,c in enumerate(Bl)}; Bset[lo]=-1
        # helpers seeded at time 0 (when A starts its extension at lo): cloud k at lo + k*step_k*CH
        helpers=[]
        for k in range(1,clouds+1):
            for j in range(members):
                st=lo+k*step_k*CH+j*spacing
                hc=chain(st,160)
                # helper reaches B at its step M (time M), index of first cut in B
                M=next((m for m,c in enumerate(hc) if c in Bset), None)
                helpers.append((hc,M))
        # map cut -> (helper, its step)
        hmap={}
        for hi,(hc,M) in enumerate(helpers):
            if M is None: continue
            for m,c in enumerate(hc[:M+1]):
                hmap.setdefault(c,(hi,m))
        done=D
        for i,c in enumerate(A[:D+1]):
            if c in hmap:
                hi,m=hmap[c]; M=helpers[hi][1]
                done=min(done, max(i, M))
                break
        out.append((D,done))
    o=np.array(out)
    print(f'clouds={clouds} members={members} spacing={spacing} every {step_k} chunks: max D {o[:,0].max()} -> completion max {o[:,1].max()} mean {o[:,1].mean():.1f} (helpers {clouds*members} per long seam)')
