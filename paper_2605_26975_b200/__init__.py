"""paper_2605_26975_b200 -- B200-native hot path of p-spectral clustering on the Grassmann manifold
(arxiv 2605.26975).  The product is libplp.so (C ABI in include/plp.h, sm_100a CUDA kernels in
csrc/); `plp` is its thin ctypes binding and `dist` the multi-GPU plumbing (torch.distributed).

The binding is imported on first use (`from paper_2605_26975_b200 import plp`), so that `build`
can run before libplp.so exists; importing `plp` without the library raises (no CPU fallback)."""

__all__ = ["plp", "dist", "build"]
