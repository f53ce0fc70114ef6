// Engine instantiation unit (see engine_impl.cuh): float 256x256
#include "engine_impl.cuh"

DCSC_ENGINE_INSTANTIATE(float, 256, 256)
