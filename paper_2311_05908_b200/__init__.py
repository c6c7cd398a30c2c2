"""B200-native FlashFFTConv hot path (arXiv 2311.05908).

The product is the C-ABI library libfftconv.so (include/fftconv.h) built from
csrc/ for sm_100a; ``fftconv`` is its thin PyTorch binding.  Importing the
binding requires the built library -- there is no CPU fallback.
"""
__all__ = ["FFTConvPlan", "launch_count_reset"]


def __getattr__(name):
    if name in __all__:
        from . import fftconv
        return getattr(fftconv, name)
    raise AttributeError(name)
