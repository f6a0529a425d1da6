import numpy as np, sys, os
sys.path.insert(0, '.')
import paper_1312_6182_b200 as gps, oracle
for (p,n,m) in [(8192,20000,64),(4096,30000,32),(2048,5000,16)]:
    rng=np.random.default_rng(1)
    A32=rng.standard_normal((p,n)).astype(np.float32); A=gps.DataMatrix(A32)
    Q,_=np.linalg.qr(rng.standard_normal((p,m))); X=Q
    gamma=np.full(m,2.0); mu=np.linspace(1,.6,m)
    A64=A32.astype(np.float64); C=A64.T@X
    G_ref=oracle.block_gradient(A64,C,gamma,mu,'l1'); f_ref=oracle.block_objective(C,gamma,mu,'l1')
    f=gps.objective_bl1(A,X,gamma,mu); G=gps.ascent_direction_block(A,X,gamma,mu,'l1')
    print(p,n,m,'seg',os.environ.get('GPSPCA_TC_SEG','def'),'f rel %.2e'%abs(f/f_ref-1),'G rel %.2e'%(np.abs(G-G_ref).max()/np.abs(G_ref).max()))
