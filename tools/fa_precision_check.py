import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth, oracle
import paper_1812_01108_b200 as tpl
oracle.build()
table = synth.load_residue_table(); tables = tpl.Tables(table)
for B, L in ((64, 700), (32, 1000), (512, 500)):
    ang = synth.angles_uniform(B, L, 8, 77); rt = synth.restype_uniform(B, L, 20, 78)
    ln = torch.full((B,), L, dtype=torch.int32)
    c = tpl.fullatom(ang.cuda(), rt.cuda(), ln.cuda(), tables).cpu().numpy()
    idx = np.arange(min(B, 64))
    X, nat = oracle.fullatom_forward(table, synth.numpy64(ang)[idx], rt.numpy()[idx], ln.numpy()[idx], c.shape[1])
    errs = [np.abs(c[b, :nat[n]] - X[n, :nat[n]]).max() for n, b in enumerate(idx)]
    print(f"FA B={B} L={L}: max coord err over {len(idx)} chains {max(errs):.3e}  median {np.median(errs):.3e}")
