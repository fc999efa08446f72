"""Ad-hoc first-light check: GPU vs oracle on c1 (developer script)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_1812_06635_b200 import _abi, fastl1 as F, synthetic as syn

orc = F.Backend(_abi.Library(Path(__file__).resolve().parents[1] / 'oracle/_build/libfl1oracle.so', 'orc_', extra=_abi.ORACLE_ONLY))
gpu = F.default_backend()
names = sys.argv[1:] or ['c1']
dense_names = [x for x in names if x.startswith('c')]
for name in dense_names:
    inst = syn.dense_instance(name)
    res = {}
    for tag, B in (('gpu', gpu), ('orc', orc)):
        d = F.DenseDictionary(inst.a, backend=B)
        # utility checks
        r = np.random.default_rng(0).standard_normal(inst.a.shape[0])
        xx = np.random.default_rng(1).standard_normal(inst.a.shape[1])
        adj = d.apply_adjoint(r); ap = d.apply(xx)
        print(tag, 'adj err', np.max(np.abs(adj - inst.a.T @ r)), 'apply err', np.max(np.abs(ap - inst.a @ xx)))
        t = time.time(); L = F.lipschitz_bound(d); tl = time.time() - t
        print(tag, 'L', repr(L), 'time', tl)
        seq = F.ApproxSequence([F.make_exact_approx(d)])
        cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
        opts = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L])
        t = time.time(); out = F.run_lasso(seq, inst.y, inst.lam, cfg, opts); el = time.time() - t
        res[tag] = out
        print(tag, name, 'conv', out.converged, 'it', out.iterations, 'gap', out.final_gap, 'S', out.final_active.size,
              'wall', el, 'dev_ms', out.device_ms, 'setup_ms', out.setup_ms, 'power', out.power_iterations, 'launches', out.kernel_launches)
        if out.profile is not None:
            pr = out.profile
            print('   profile ms: A %.3f  B %.3f  D %.3f  power %.3f  switch %.3f ; A^T r bytes %.3g -> %.1f GB/s' % (pr[0]/1e6, pr[1]/1e6, pr[2]/1e6, pr[3]/1e6, pr[4]/1e6, pr[5], pr[5]/pr[0] if pr[0] else 0))
    g, o = res['gpu'], res['orc']
    print('x maxdiff', np.max(np.abs(g.x - o.x)), 'support equal', np.array_equal(g.x != 0, o.x != 0))
    print('trace active equal', np.array_equal(g.trace['active_size'], o.trace['active_size']),
          'nnz equal', np.array_equal(g.trace['x_nnz'], o.trace['x_nnz']), 'flops equal', np.array_equal(g.trace['flops_cum'], o.trace['flops_cum']))
    gg, og = g.trace['gap'], o.trace['gap']
    print('gap rel diff max', np.max(np.abs(gg - og) / np.maximum(np.abs(og), 1e-300)))

# SuKro operator checks (small) + C3-style solve at reduced size
if 'sukro' in names:
    rng = np.random.default_rng(7)
    m, q, T = 8, 12, 3
    lefts = [rng.standard_normal((m, q)) for _ in range(T)]
    rights = [rng.standard_normal((m, q)) for _ in range(T)]
    scale = rng.uniform(0.5, 2.0, q * q)
    dense = syn.kron_dense(lefts, rights, scale)
    for tag, B in (('gpu', gpu), ('orc', orc)):
        S = F.SukroDictionary(list(zip(lefts, rights)), col_scale=scale, backend=B)
        x = rng.standard_normal(q * q); r = rng.standard_normal(m * m)
        print(tag, 'sukro apply err', np.max(np.abs(S.apply(x) - dense @ x)), 'adj err', np.max(np.abs(S.apply_adjoint(r) - dense.T @ r)),
              'col err', np.max(np.abs(S.column(5) - dense[:, 5])), 'norms err', np.max(np.abs(S.atom_norms2() - np.linalg.norm(dense, axis=0))))
        print(tag, 'L', F.lipschitz_bound(S), 'ref', 1.05 * np.linalg.norm(dense, 2) ** 2)
    inst = syn.sukro_instance(seed=3, m=16, q=32, terms=6, levels=(1, 2, 4), nnz=30)
    res = {}
    for tag, B in (('gpu', gpu), ('orc', orc)):
        levels = []
        for li, nt in enumerate(inst.levels):
            op = F.SukroDictionary(list(zip(inst.lefts[:nt], inst.rights[:nt])), col_scale=inst.col_scale, backend=B)
            levels.append(F.ApproxDictionary(op, inst.eps[li], float(inst.eps[li].max()), inst.rc[li], inst.approx_norms[li], inst.exact_norms))
        ex = F.DenseDictionary(inst.a, backend=B)
        levels.append(F.make_exact_approx(ex))
        seq = F.ApproxSequence(levels)
        cfg = F.SwitchConfig(screening_interval=10, max_iterations=20000, rel_tolerance=1e-6, gamma_threshold=0.5)
        out = F.run_lasso(seq, inst.y, inst.lam, cfg, F.RunOptions())
        res[tag] = out
        print(tag, 'c3-small conv', out.converged, 'it', out.iterations, 'gap', out.final_gap, 'switches', out.switches.tolist(), 'dev_ms', out.device_ms)
    g, o = res['gpu'], res['orc']
    print('x maxdiff', np.max(np.abs(g.x - o.x)), 'support equal', np.array_equal(g.x != 0, o.x != 0),
          'trace active equal', np.array_equal(g.trace['active_size'], o.trace['active_size']),
          'dict idx equal', np.array_equal(g.trace['dict_index'], o.trace['dict_index']))
