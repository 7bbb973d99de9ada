"""B200-native (sm_100a) hash-grid INR library for arXiv 2304.10516's
distributed neural representation: the fit + decode hot path behind the C ABI
of include/inr.h (libinr.so), with a thin ctypes binding (`inr`) and the
multi-GPU shell (`dnr`, torch.distributed for process groups only)."""
