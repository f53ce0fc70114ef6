// Engine instantiation unit (see engine_impl.cuh): double / float 48x48, float 80x80
#include "engine_impl.cuh"

DCSC_ENGINE_INSTANTIATE(double, 48, 48)
DCSC_ENGINE_INSTANTIATE(float, 48, 48)
DCSC_ENGINE_INSTANTIATE(float, 80, 80)
