import sys, numpy as np
sys.path.insert(0, '.')
import paper_1505_04650_b200 as C
from oracle import cnmf_oracle as O
g = np.load('tests/golden/reference_vectors.npz')
a = g['cmp_a']
for w in (0, 1, 2):
    cfg = C.CompressionConfig(r=8, r_ov=12, w=w, seed=3)
    q = C.structured_compress(a, cfg).Q
    ref = O.range_basis(a, O.Config(8, 12, w, 3), reorth=True)
    print('w', w, 'orth', np.linalg.norm(q.T @ q - np.eye(20)), 'pd', O.projector_distance(q, ref),
          'colmax', [float('%.2e' % np.abs(q[:, j] - ref[:, j]).max()) for j in range(0, 20, 3)],
          'resid', O.residual_norm(a, q), O.residual_norm(a, ref))
    qr_ = C.structured_compress_rows(a, cfg).Q
    refr = O.row_basis(a, O.Config(8, 12, w, 3), reorth=True)
    print('   rows orth', np.linalg.norm(qr_.T @ qr_ - np.eye(20)), 'pd', O.projector_distance(qr_, refr))
a = O.dense_lowrank(2000, 1000, 20, 0.01, seed=0)
for side in (0, 1):
    for w in (0, 1, 4):
        cfg = C.CompressionConfig(r=20, r_ov=10, w=w, seed=5)
        q = (C.structured_compress if side == 0 else C.structured_compress_rows)(a, cfg).Q
        ref = (O.range_basis if side == 0 else O.row_basis)(a, O.Config(20, 10, w, 5), reorth=True)
        aa = a if side == 0 else a.T
        print('lowrank side', side, 'w', w, 'orth', np.linalg.norm(q.T @ q - np.eye(30)), 'pd', O.projector_distance(q, ref),
              'resid', O.residual_norm(aa, q), O.residual_norm(aa, ref))
