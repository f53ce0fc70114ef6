// Engine instantiation unit (see engine_impl.cuh): float 100x100
#include "engine_impl.cuh"

DCSC_ENGINE_INSTANTIATE(float, 100, 100)
