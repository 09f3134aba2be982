"""Per-IPM-iteration trace (μ, residual norms, α, PCG iterations) of the library's IPM."""
import sys
sys.path.insert(0, '.')
import qpgen
from paper_2104_12916_b200.binding import from_qp
name, prec = sys.argv[1], sys.argv[2]
maxit = int(sys.argv[3]) if len(sys.argv) > 3 else 2000
n_it = int(sys.argv[4]) if len(sys.argv) > 4 else 30
space = sys.argv[5] if len(sys.argv) > 5 else "nu"
qp = qpgen.make(name)
s = from_qp(qp)
s.ipm_factor_once(prec)
s.ipm_init(ipm_tol=1e-8, max_ipm=100, pcg_maxit=maxit, space=space)
for k in range(n_it):
    r = s.ipm_iterate(1)
    D, rnu, eps = s.ipm_last_system()
    print(f"{k:3d} mu {r['mu']:.3e} rg {r['rg_inf']:.2e} re {r['re_inf']:.2e} ri {r['ri_inf']:.3e} alpha {r['alpha']:.4f} "
          f"pcg {r['pcg_iters'][-1] if r['pcg_iters'] else 0} eps {eps:.1e} Dmin {D.min():.2e} Dmax {D.max():.2e}",
          flush=True)
    if r['converged']:
        print('converged'); break
