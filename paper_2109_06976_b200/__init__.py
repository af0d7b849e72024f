"""B200-native batched rigid-body dynamics with analytical gradients.

A from-scratch sm_100a implementation of the GRiD path (arXiv 2109.06976):
ID (RNEA), direct Minv, FD, dID and dFD per trajectory knot point, generated
per robot as straight-line CUDA and exposed through the reference package's
API (`rbdgen`): `urdf.parse_urdf`, `models.load`, the refdyn-style functions
in `dynamics` (with f_ext), the operator pair `program.build` /
`program.interpret`, device-resident rollouts (`rollout`), the reference's
kernel text format (`kdump`) and the spec CLI (`python -m ...cli`).
"""

from . import codegen, dynamics, kdump, kernels, models, program, rollout, runtime, schedule, spatial, urdf
from .dynamics import (DynamicsGradients, bias_force, fd_grad, forward_dynamics, minv_direct,
                       rnea, rnea_grad)
from .models import load
from .program import InterpreterError, build, interpret
from .urdf import parse_urdf

__all__ = ["codegen", "dynamics", "kdump", "kernels", "models", "program", "rollout", "runtime", "schedule",
           "spatial", "urdf", "DynamicsGradients", "bias_force", "fd_grad", "forward_dynamics",
           "minv_direct", "rnea", "rnea_grad", "load", "InterpreterError", "build", "interpret",
           "parse_urdf"]
