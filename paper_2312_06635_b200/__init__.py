"""B200-native chunk-wise Gated Linear Attention (arXiv 2312.06635): CUDA kernels for sm_100a behind a C ABI
(include/gla.h, libgla.so) plus this thin binding.  See DESIGN.md."""
from .binding import (GLAError, GLAFunction, chunk_bwd, chunk_fwd, dstate_summary, gla, lib, recurrent_step,
                  resolve_path, state_combine, state_summary)

__all__ = ["GLAError", "GLAFunction", "chunk_bwd", "chunk_fwd", "dstate_summary", "gla", "lib", "recurrent_step",
           "resolve_path", "state_combine", "state_summary"]
