"""Device error metric for the non-central chi-squared tables (metrics.py:300-350).

``rmse_ncchi2(tables, lambda_grid, n_samples)`` regenerates the paper's Table 5
RMSE grid on the GPU: for each (table, lambda) the midpoint lattice
u_i = (i + 1/2)/n is mapped through the table (``ncchi2_eval``, shared lambda)
and through the exact quantile (device safeguarded Newton, warm-started from
the table, residual contract |F - u| <= tol_f), and the RMSE of the
difference is reduced on the device.  Cells whose exact quantile misses the
1e-8 residual contract are NaN and listed in ``failures`` like the reference.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as dev
from . import _kernels as kernels
from ._native import call
from .tables import NcChi2Table


@dataclass
class RmseGrid:
    nus: list
    lambdas: list
    values: np.ndarray  # (len(lambdas), len(nus)); NaN marks failed cells
    n_samples: int
    failures: list = field(default_factory=list)


def exact_ncchi2_quantiles(u: torch.Tensor, nu: float, lam: float, x0: torch.Tensor | None = None):
    """(x, |F(x) - u|) for a shared lambda on the device."""
    ld = torch.full((1,), float(lam), dtype=torch.float64, device=u.device)
    x = torch.empty_like(u)
    r = torch.empty_like(u)
    call("arv_ncchi2_inv_cdf", u.data_ptr(), ld.data_ptr(), 1, float(nu), x0.data_ptr() if x0 is not None else None,
         x.data_ptr(), r.data_ptr(), u.numel(), dev.stream_handle(u.device))
    return x, r


def rmse_ncchi2(tables, lambda_grid, n_samples: int = 10**5) -> RmseGrid:
    if isinstance(tables, NcChi2Table) or type(tables).__name__ == "NcChi2Table":
        tables = [tables]
    device = dev.require_cuda()
    lambdas = [float(x) for x in lambda_grid]
    values = np.full((len(lambdas), len(tables)), np.nan)
    failures = []
    u = (torch.arange(n_samples, dtype=torch.float64, device=device) + 0.5) / n_samples
    for cj, table in enumerate(tables):
        for ri, lam in enumerate(lambdas):
            xa = torch.empty_like(u)
            kernels.ncchi2_eval(table.eval_stacks, table.nu, u, torch.full((1,), lam, dtype=torch.float64,
                                                                            device=device), xa)
            xe, resid = exact_ncchi2_quantiles(u, table.nu, lam, x0=xa)
            worst = float(resid.max())
            if not worst <= 1e-8:
                failures.append({"nu": table.nu, "lambda": lam, "error": f"worst residual {worst:.3g}"})
                continue
            values[ri, cj] = math.sqrt(float(torch.mean((xa - xe) ** 2)))
    return RmseGrid(nus=[t.nu for t in tables], lambdas=lambdas, values=values, n_samples=n_samples,
                    failures=failures)
