import sys; sys.path.insert(0,'.')
import qpgen
from paper_2104_12916_b200.binding import from_qp
qp=qpgen.make(sys.argv[1]); s=from_qp(qp); s.ipm_factor_once('high'); print(s.stats()['nnz_LPH'])
