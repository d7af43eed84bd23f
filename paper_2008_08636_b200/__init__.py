"""B200-native weighted-level sweep of ParDNN (arXiv 2008.08636).

The compute path is libpdnn.so (hand-written sm_100a CUDA behind the C ABI in
include/pdnn.h); this package is its thin Python binding.  Importing the
package does not load the library; the first call does, and fails loudly if
it is missing (there is no CPU fallback).
"""
import importlib

__all__ = ["Graph", "PdnnError", "load_library", "EVAL_RESULT_DTYPE"]


def __getattr__(name):
    if name.startswith("__"):
        raise AttributeError(name)
    mod = importlib.import_module(__name__ + "._binding")
    if hasattr(mod, name):
        return getattr(mod, name)
    raise AttributeError(name)
