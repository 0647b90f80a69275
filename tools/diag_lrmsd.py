import numpy as np, sys, torch
sys.path.insert(0,'.')
import synth, oracle
from oracle import lrmsd as OL
from paper_1812_01108_b200 import _abi
B,L,noise=4,700,0.05
ang = synth.angles_uniform(B, L, 3, 51 + L)
ln = torch.full((B,), L, dtype=torch.int32)
a64=synth.numpy64(ang); lnn=ln.numpy()
X = oracle.backbone_forward(a64, lnn)
rng = np.random.default_rng(52)
q = rng.standard_normal(4); q /= np.linalg.norm(q)
Y = X @ OL.rotation(q).T + np.array([5.0, -3.0, 2.0]) + noise * rng.standard_normal(X.shape)
target = torch.tensor(Y, dtype=torch.float32); Y = target.numpy().astype(np.float64)
out = torch.zeros(B, device="cuda"); state = torch.zeros(B, 16, device="cuda")
g = torch.zeros(B, L, 3, device="cuda"); c = torch.zeros(B, 3*L, 3, device="cuda")
ws = torch.zeros(_abi.tpl_workspace_bytes(0, B, L), dtype=torch.uint8, device="cuda")
_abi.tpl_backbone_lrmsd_fused(ang.cuda(), ln.cuda(), target.cuda(), c, out, state, g, ws)
torch.cuda.synchronize()
cc=c.cpu().numpy().astype(np.float64); st=state.cpu().numpy(); gg=g.cpu().numpy()
for b in range(B):
    val,U,cx,cy=OL.lrmsd(cc[b],Y[b])
    Ug=st[b,:9].reshape(3,3)
    print(b,'U err',np.abs(Ug-U).max(),'cx err',np.abs(st[b,9:12]-cx).max(),'cy err',np.abs(st[b,12:15]-cy).max(),'val',out[b].item(),val, 'scale', st[b,15], 1/(3*L*val))
    _, gx = OL.batch(cc[b:b+1], Y[b:b+1], [3*L])
    G = oracle.backbone_backward(a64[b:b+1], lnn[b:b+1], gx)[0]
    err=np.abs(gg[b]-G); i=np.unravel_index(np.argmax(err),err.shape)
    print('   grad rel', err.max()/np.abs(G).max(), 'worst at', i, gg[b][i], G[i])
