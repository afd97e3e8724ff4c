"""ORACLE — test infrastructure only (see oracle/core.py header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package.  The product path (paper_1309_5050_b200) never does.
"""
from .core import (Shapes, shapes, shapes_rect, trajmat, xv, xv_rows, xtu, svd_dense, svd_gram,  # noqa: F401
                   diagsums, diagsums_cells, reconstruct, reconstruct_cells, wcorr, contributions, esprit, vector_forecast,
                   fix_signs, build)
