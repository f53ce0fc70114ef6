// Engine instantiation unit (see engine_impl.cuh): double 128x128 — the FP64
// half spectrum (133 KB) needs two plane buffers, so this grid runs on the
// 4-CTA cluster family like the FP32 256x256 one
#include "engine_impl.cuh"

DCSC_ENGINE_INSTANTIATE(double, 128, 128)
