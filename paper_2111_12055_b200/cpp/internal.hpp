// internal.hpp — shared plumbing of the drop-in's translation units (not an
// installed header): the process-wide device context and the mapping of C-ABI
// status codes onto the reference's exception types.
#pragma once

struct gbxcu_ctx;

namespace gbx::detail {

// The libgbxcu context every drop-in call uses (device 0, $GBX_DEVICE, or
// set_device()); created on first use, throws without a usable B200.
gbxcu_ctx* device_context();

// GBXCU_OK -> return; otherwise throw the reference's exception type.
void check_status(int rc, int diverged_epoch = -1);

}  // namespace gbx::detail
