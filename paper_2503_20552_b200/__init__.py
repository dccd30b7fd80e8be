"""B200-native (sm_100a) implementation of Adrenaline's offloaded decode-attention
path (arXiv 2503.20552), behind the Python API of the reference simulator
(adrenaline_sim): ``import paper_2503_20552_b200 as adrenaline_sim`` exposes the
same modules (specs, costs, calibration, scheduling, graphs, config, workload,
engine). The CUDA kernels live in libadrenaline.so (csrc/, C-ABI in
include/adrenaline.h); ``ops`` is the torch-tensor front end and ``runtime`` /
``exchange`` / ``coloc`` / ``kvcache`` the B200 runtime around it (imported on
demand: they need torch)."""

from . import calibration, config, costs, engine, graphs, scheduling, specs, workload  # noqa: F401

__version__ = "0.1.0"
