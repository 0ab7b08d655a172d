import os, sys
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
os.environ['SRT3D_FUZZ_BASE'] = '5000'
import numpy as np, torch
import paper_2203_00952_b200 as gpu, oracle, srt3d_inputs as inputs_mod
import test_gpu_fuzz as f
c = f._case(254)
T, m = c['T'], c['m']
bins, offs = inputs_mod.random_csr(npix=c['npix'], T=T, max_n=c['max_n'], seed=c['seed'])
zo = oracle.sketch(bins, offs, T, m)
db = torch.from_numpy(bins).cuda(); do = torch.from_numpy(offs).cuda()
for name, path, lanes in [('auto', gpu.PATH_AUTO, 0), ('d4', gpu.PATH_DIRECT, 4), ('d8', gpu.PATH_DIRECT, 8), ('d16', gpu.PATH_DIRECT, 16), ('d32', gpu.PATH_DIRECT, 32), ('bc', gpu.PATH_BINCOUNT, 0), ('paired', gpu.PATH_PAIRED, 0), ('tensor', gpu.PATH_TENSOR, 0)]:
    try:
        z = gpu.srt3d_sketch_ex(db, do, T, m, total_photons=int(offs[-1]), path=path, lanes_per_pixel=lanes)
    except gpu.Srt3dError as e:
        print(name, 'err', e); continue
    torch.cuda.synchronize()
    d = np.abs(z.cpu().numpy() - zo)
    i, j = np.unravel_index(np.argmax(d), d.shape)
    n = offs[i+1]-offs[i]
    print(name, f'{d.max():.3e}', 'pix', i, 'freq', j+1, 'n', n, 'bins', bins[offs[i]:offs[i+1]].tolist())

# tensor path: error distribution, repeatability, and the pass structure (m > 32: j0 = 0, 32)
zs = [gpu.srt3d_sketch_ex(db, do, T, m, total_photons=int(offs[-1]), path=gpu.PATH_TENSOR).cpu().numpy() for _ in range(3)]
print('repeat bitwise', all(np.array_equal(zs[0].view(np.uint64), z.view(np.uint64)) for z in zs[1:]))
d = np.abs(zs[0] - zo)
bad = np.argwhere(d > 2e-6)
print('n bad entries', len(bad), 'pixels', sorted(set(bad[:, 0].tolist()))[:20], 'freqs', sorted(set((bad[:, 1] + 1).tolist()))[:40])
for i in sorted(set(bad[:, 0].tolist()))[:8]:
    print(i, 'tile', i // 4, 'slot', i % 4, 'n', offs[i+1]-offs[i], 'bins', bins[offs[i]:offs[i+1]].tolist(), 'maxd', d[i].max(), 'at freq', int(np.argmax(d[i])) + 1)
for mm in (32, 16, 30):
    z2 = gpu.srt3d_sketch_ex(db, do, T, mm, total_photons=int(offs[-1]), path=gpu.PATH_TENSOR).cpu().numpy()
    print('m', mm, 'maxd', np.abs(z2 - oracle.sketch(bins, offs, T, mm)).max())
