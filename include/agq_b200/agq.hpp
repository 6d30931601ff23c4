// Umbrella header of the B200 drop-in: the reference's agq:: API
// (quantize, fp8, tensor_io, collective, dbca policy) backed by the sm_100a
// kernels of libagq_cuda.so. Swap `-I<reference>/proj/include` +
// `#include "agq/quantize.hpp"` for `-I<repo>/include` +
// `#include "agq_b200/quantize.hpp"` and link `-lagq_cuda`.
#pragma once
#include "collective.hpp"
#include "dbca.hpp"
#include "fp8.hpp"
#include "quantize.hpp"
#include "tensor_io.hpp"
