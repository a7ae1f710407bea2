"""Interface factorisation work, a face-level symbolic model.

Nodes are faces (q unknowns each); elimination cost of a node with front F (unknowns) is
q^3/3 + q^2 F + q F^2; nested dissection by recursive bisection of the P x P subdomain grid.
  "M":   the Schur matrix of eqn:schur, M = S1 + Q^T Q -- Q^T Q couples the faces of two adjacent
         subdomains, so a separator must hold every face touching one subdomain column (3 faces
         per row); this is the order the tile Cholesky uses (reading R25).
  "aug": the quasi-definite augmented system [S1 Q^T; Q -I] [u; lambda] (lambda = the flux
         residual): a separator is one line of faces (u and lambda), half the flops -- but S1 alone
         is nearly singular (the local networks fit smooth boundary data almost exactly), so an
         LDL^T in the nested-dissection order has unbounded growth: not usable.
usage: python tools/iface_flops.py P q
"""
import sys
from collections import defaultdict

P=int(sys.argv[1]); q=int(sys.argv[2])
# faces: V(i,j) i<P-1 (between (i,j),(i+1,j)), H(i,j) j<P-1 (between (i,j),(i,j+1))
faces={}
def fid(key):
    if key not in faces: faces[key]=len(faces)
    return faces[key]
def sub_faces(i,j):
    out=[]
    if i>0: out.append(('V',i-1,j))
    if i<P-1: out.append(('V',i,j))
    if j>0: out.append(('H',i,j-1))
    if j<P-1: out.append(('H',i,j))
    return out
allf=[('V',i,j) for j in range(P) for i in range(P-1)]+[('H',i,j) for j in range(P-1) for i in range(P)]
def subs_of(f):
    t,i,j=f
    return [(i,j),(i+1,j)] if t=='V' else [(i,j),(i,j+1)]
def pos(f):  # face center coordinates in units of subdomain
    t,i,j=f
    return (i+1, j+0.5) if t=='V' else (i+0.5, j+1)
# graph 1: M = S1 + Q^T Q
def graph_M():
    nodes=[('u',f) for f in allf]
    adj=defaultdict(set)
    for i in range(P):
        for j in range(P):
            fs=sub_faces(i,j)
            for a in fs:
                for b in fs: adj[('u',a)].add(('u',b))
    for f in allf:
        A,B=subs_of(f); fs=set(sub_faces(*A))|set(sub_faces(*B))
        for a in fs:
            for b in fs: adj[('u',a)].add(('u',b))
    return nodes,adj
def graph_aug():
    nodes=[('u',f) for f in allf]+[('l',f) for f in allf]
    adj=defaultdict(set)
    for i in range(P):
        for j in range(P):
            fs=sub_faces(i,j)
            for a in fs:
                for b in fs: adj[('u',a)].add(('u',b))
    for f in allf:
        A,B=subs_of(f); fs=set(sub_faces(*A))|set(sub_faces(*B))
        adj[('l',f)].add(('l',f))
        for a in fs:
            adj[('l',f)].add(('u',a)); adj[('u',a)].add(('l',f))
    return nodes,adj
def nd_order(nodes, adj, sepfun):
    order=[]
    def rec(ns, box, depth):
        x0,x1,y0,y1=box
        if len(ns)<=8 or (x1-x0<=1 and y1-y0<=1):
            order.extend(sorted(ns,key=lambda n:(pos(n[1]),n[0]))); return
        if x1-x0>=y1-y0:
            c=(x0+x1)//2; axis=0
        else:
            c=(y0+y1)//2; axis=1
        sep,left,right=sepfun(ns,c,axis)
        lb=(x0,c,y0,y1) if axis==0 else (x0,x1,y0,c)
        rb=(c,x1,y0,y1) if axis==0 else (x0,x1,c,y1)
        rec(left,lb,depth+1); rec(right,rb,depth+1)
        order.extend(sep)
    rec(nodes,(0,P,0,P),0)
    return order
def sep_M(ns,c,axis):
    # faces touching subdomain column/row c (subdomains with index c along axis)... use faces touching column c
    sep=[];L=[];R=[]
    for n in ns:
        f=n[1]; ss=subs_of(f)
        if any(s[axis]==c for s in ss): sep.append(n)
        elif pos(f)[axis]<c: L.append(n)
        else: R.append(n)
    return sep,L,R
def sep_aug(ns,c,axis):
    sep=[];L=[];R=[]
    for n in ns:
        f=n[1]; p=pos(f)[axis]
        if p==c and ((f[0]=='V')==(axis==0)): sep.append(n)
        elif p<c: L.append(n)
        else: R.append(n)
    return sep,L,R
def cost(nodes,adj,order):
    idx={n:k for k,n in enumerate(order)}
    # symbolic elimination at node (block) level
    struct={n:set(m for m in adj[n] if idx[m]>idx[n]) for n in nodes}
    fl=0.0; nnzL=0
    for n in order:
        s=struct[n]
        F=len(s)*q
        fl+= q**3/3 + q*q*F + q*F*F
        nnzL+= q*q/2+q*F
        if s:
            par=min(s,key=lambda m:idx[m])
            struct[par] |= (s-{par})
    return fl, nnzL
for name,g,sf in [("M",graph_M,sep_M),("aug",graph_aug,sep_aug)]:
    nodes,adj=g()
    o=nd_order(nodes,adj,sf)
    assert len(o)==len(nodes) and len(set(o))==len(nodes)
    fl,nnz=cost(nodes,adj,o)
    print(name, len(nodes)*q, "flop %.3e"%fl, "nnzL %.3e"%nnz)
