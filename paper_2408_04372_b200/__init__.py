"""B200-native space-time multigrid (STMG) solve path of arXiv 2408.04372:
fused fp64 space-time operator, exact cell-wise space-time additive Schwarz
smoother, h/p/tau/k transfers, coarse solve and device-resident GMRES, all
behind the C ABI in include/stmg_b200.h (libstmg_b200.so, sm_100a)."""
from .api import (ASMSmoother, Mesh, SpaceTimeMultigrid, SpaceTimeOperator, Transfer, gmres, gmres_options,
                  mg_options)
from . import problems

__all__ = ["Mesh", "SpaceTimeOperator", "ASMSmoother", "Transfer", "SpaceTimeMultigrid", "gmres", "gmres_options",
           "mg_options", "problems"]
