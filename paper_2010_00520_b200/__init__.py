"""paper_2010_00520_b200 -- B200 (sm_100a) FMM-FFT translation stage with
compressed FFT'ed translation operators (arXiv 2010.00520).

The product is the C-ABI library libfmmt.so (include/fmmt.h, sources in
csrc/); `fmmt` is its thin Python binding.  PyTorch is used by callers only
for device memory, streams and torch.distributed.
"""
__all__ = ["fmmt", "build"]
