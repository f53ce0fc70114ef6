// Engine instantiation unit (see engine_impl.cuh): double 16x20, float 16x20
#include "engine_impl.cuh"

DCSC_ENGINE_INSTANTIATE(double, 16, 20)
DCSC_ENGINE_INSTANTIATE(float, 16, 20)
