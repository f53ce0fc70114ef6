// Engine instantiation unit (see engine_impl.cuh): float 128x128
#include "engine_impl.cuh"

DCSC_ENGINE_INSTANTIATE(float, 128, 128)
