// sfi_b200.hpp — umbrella header of the C++ host API.
//
// The API itself is the reference's operator interface under the reference's
// own header paths and namespace (include/sfi/*.hpp, namespace sfi: same
// types, field layouts, signatures, defaults and error codes as
// /root/reference/proj/include/sfi/*.hpp), so a reference caller recompiles
// and relinks against libsfi_b200.so unchanged. Every hot-path call launches
// the sm_100a kernels through the C ABI (sfi_b200.h); there is no CPU
// fallback. B200 extensions (DeviceCache, dense_capture, KvStore prefill /
// device accessors, check, the DecodeExecutor of sfi/decode.hpp) live beside
// them in namespace sfi.
//
// `sfi_b200` is kept as an alias of `sfi` for existing callers.
#pragma once

#include "sfi_b200.h"
#include "sfi/attention.hpp"
#include "sfi/config.hpp"
#include "sfi/decode.hpp"
#include "sfi/distribution.hpp"
#include "sfi/error.hpp"
#include "sfi/scheduler.hpp"
#include "sfi/selector.hpp"

namespace sfi_b200 = sfi;
