"""B200-native MOREA hot path: batched objective evaluation of dual-dynamic
tetrahedral-mesh deformations (arXiv 2303.04873) behind the C-ABI in
include/morea.h.  `morea` is the ctypes binding; `distributed` shards a
population over ranks."""
