import numpy as np, torch, sys
sys.path.insert(0,'.')
import oracle, synth
from tests import ecref
from paper_2504_14497_b200 import pcmm as P
sk, pk = P.keygen(5)
x = int.from_bytes(sk,'big')
b = np.array([3, 0, 7], dtype=np.int64)
r = synth.scalars_to_be_bytes([11, 12, 13])
ct = oracle.encrypt(pk, b, r)
m, st = P.decrypt_small(sk, torch.from_numpy(ct).cuda(), 0, 10)
print('dec', m.cpu().numpy(), st.cpu().numpy())
# recompute M via hooks
C1 = torch.from_numpy(ct[:, :64].copy()).cuda(); C2 = torch.from_numpy(ct[:, 64:].copy()).cuda()
K = torch.from_numpy(np.frombuffer(b''.join(((ecref.Q - x)).to_bytes(32,'big')+bytes(32) for _ in range(3)),dtype=np.uint8).reshape(3,64).copy()).cuda()
nx = P.test_point(3, C1, K)
M = P.test_point(0, C2, nx).cpu().numpy()
for i in range(3): print(i, M[i].tobytes() == ecref.mulG(int(b[i])))
