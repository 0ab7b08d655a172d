import os, sys
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
os.environ['SRT3D_FUZZ_BASE'] = '5000'
import numpy as np, torch
import paper_2203_00952_b200 as gpu, oracle, srt3d_inputs as inputs_mod
import test_gpu_fuzz as f
c = f._case(254)
T, m = c['T'], 32
bins, offs = inputs_mod.random_csr(npix=c['npix'], T=T, max_n=c['max_n'], seed=c['seed'])
def run(lists, label):
    b = np.concatenate([np.array(l, dtype=np.uint16) for l in lists]) if sum(len(l) for l in lists) else np.zeros(0, np.uint16)
    o = np.zeros(len(lists) + 1, dtype=np.uint32); o[1:] = np.cumsum([len(l) for l in lists])
    db = torch.from_numpy(b).cuda() if b.size else torch.zeros(1, dtype=torch.uint16, device='cuda')
    z = gpu.srt3d_sketch_ex(db, torch.from_numpy(o).cuda(), T, m, total_photons=int(o[-1]), path=gpu.PATH_TENSOR).cpu().numpy()
    zo = oracle.sketch(b, o, T, m)
    d = np.abs(z - zo)
    print(label, f'{d.max():.3e}', 'per pixel', [f'{x:.1e}' for x in d.max(1)][:8])
L = [bins[offs[i]:offs[i+1]].tolist() for i in range(len(offs) - 1)]
run([L[2436]], 'alone')
run(L[2436:2440], 'its tile')
run(L[2432:2444], '3 tiles')
run([[17], [1943]], 'split')
run([[17, 1943]], 'pair')
run([[1943, 17]], 'pair rev')
run([[17, 1943]] * 8, 'pair x8')
print('tile 609 pixels', L[2436:2440])
