// Engine instantiation unit (see engine_impl.cuh): double 20x20, float 20x20
#include "engine_impl.cuh"

DCSC_ENGINE_INSTANTIATE(double, 20, 20)
DCSC_ENGINE_INSTANTIATE(float, 20, 20)
