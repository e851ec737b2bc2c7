import sys, numpy as np
sys.path.insert(0, '.')
import paper_1505_04650_b200 as C
from oracle import cnmf_oracle as O
for rows, cols, seed in [(20000, 60, 7), (9000, 30, 2**63 + 1), (4096, 60, 7)]:
    cfg = C.CompressionConfig(r=cols, r_ov=0, w=0, seed=seed)
    got = C.draw_test_matrix(cfg, rows).cpu().numpy()
    want = O.test_matrix(rows, cols, seed)
    bad = np.argwhere(got != want)
    print(rows, cols, seed, 'mismatches', len(bad), bad[:5].tolist())
    if len(bad):
        flat = got.ravel(); wf = want.ravel(); k = np.flatnonzero(flat != wf)
        print(' first flat idx', k[:10], 'chunk-local', [(i // cols) % 4096 * cols + i % cols for i in k[:10]])
        print(' got', flat[k[:4]], 'want', wf[k[:4]])
        # is it a shift?
        i = k[0]
        print(' got[i] in want near?', [j for j in range(i-5, i+6) if j < len(wf) and wf[j] == flat[i]])
