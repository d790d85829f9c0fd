"""Third-party reference definitions used as pins (not our code).

``to_blocked`` is torch's own definition of the cuBLASLt block-scaling-factor
layout (torch/testing/_internal/common_quantized.py, which cites the cuBLAS docs
"d-block-scaling-factors-layout").  Importing that module needs ``expecttest``
(absent here), so the two functions are lifted from its source with ``ast``.
"""
import ast
import os

import torch

_SRC = os.path.join(os.path.dirname(torch.__file__), "testing", "_internal", "common_quantized.py")


def _load(names):
    tree = ast.parse(open(_SRC).read())
    fns = [n for n in tree.body if isinstance(n, ast.FunctionDef) and n.name in names]
    mod = ast.Module(body=fns, type_ignores=[])
    ns = {"torch": torch}
    exec(compile(mod, _SRC, "exec"), ns)
    return ns


_ns = _load({"to_blocked", "ceil_div"})
to_blocked = _ns["to_blocked"]
