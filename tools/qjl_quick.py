import sys; sys.path.insert(0, '.')
import numpy as np, torch, iqsynth
import paper_2603_28430_b200 as iq
from oracle import qjl_oracle as Q, iq_oracle as O
d=128; p=iq.iq_make_params_qjl(d,3,iq.FULL,iqsynth.PARAMS_SEED,device=0)
X=iqsynth.unit_vectors(300,d,5,np.float16)
x=torch.from_numpy(X).cuda()
codes,norms,qjl,rn=iq.iq_quantize_qjl(p,x); torch.cuda.synchronize()
print("ran", qjl[:2].cpu().numpy(), rn[:4].cpu().numpy())
S=Q.sketch_matrix(d, iqsynth.PARAMS_SEED); po=O.make_params(d,3,O.FULL,iqsynth.PARAMS_SEED)
c,pk,rho,xh,q,g=Q.encode(X,po,S)
bg=Q.unpack_bits(qjl.cpu().numpy(),d)
print("agree", (bg==q).mean(), "gamma rel", np.max(np.abs(rn.cpu().numpy()-g)/g))
