"""B200-native (sm_100a) implementation of Adrenaline's offloaded decode-attention
path (arXiv 2503.20552), behind the Python API of the reference simulator
(adrenaline_sim). The CUDA kernels live in libadrenaline.so (csrc/, C-ABI in
include/adrenaline.h); ``ops`` is the torch-tensor front end."""

__version__ = "0.1.0"
