// Engine instantiation unit (see engine_impl.cuh): double 64x64
#include "engine_impl.cuh"

DCSC_ENGINE_INSTANTIATE(double, 64, 64)
