// Engine instantiation unit (see engine_impl.cuh): float 64x64
#include "engine_impl.cuh"

DCSC_ENGINE_INSTANTIATE(float, 64, 64)
