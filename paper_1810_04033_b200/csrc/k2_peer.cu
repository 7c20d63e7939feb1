// k2_peer.cu — the streaming pass kernels instantiated with the slab runner's
// peer stores (sl_sweep_pass_peer).  A separate translation unit so the two
// sets of instantiations compile in parallel; the plain passes carry no
// peer-store code at all.
#define SL_PEER_TU
#include "k2_fused.cu"
