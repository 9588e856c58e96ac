import sys, os, numpy as np
sys.path.insert(0,'.')
from oracle.oracle import Oracle
o=Oracle()
T,S=int(sys.argv[1]),int(sys.argv[2])
q=o.generate(1,T,S,0)[0]
Q=o.forward_parallel(q)
bits=np.zeros((T,S),bool); bits[1:,:]=Q[:-1,:]>Q[1:,:]
print("bit density", bits[1:].mean())
L=256
for k in [2, 10, 20, 28]:
    hi=(k+1)*L; lo=k*L
    pos=np.arange(T)
    distinct=[]
    for j in range(hi-1, lo-1, -1):
        mv=(pos>0)&bits[pos,j]
        pos=pos-mv
        if (hi-1-j) in (0,16,32,64,128,255): distinct.append((hi-1-j, len(np.unique(pos))))
    print("segment",k,"distinct walkers after cols:",distinct)
