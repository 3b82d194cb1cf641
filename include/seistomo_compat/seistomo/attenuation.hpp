// seistomo/attenuation.hpp (reference: proj/core/include/seistomo/attenuation.hpp) -> the B200
// drop-in. Put include/seistomo_compat on the include path instead of the
// reference's include/ to build a seistomo caller against libhz_b200.so.
#pragma once
#ifndef HZ_B200_AS_SEISTOMO
#define HZ_B200_AS_SEISTOMO
#endif
#include "../../hz_b200.hpp"
