// gqsa_pack_internal.h -- LAYOUT-TC entry points shared by gqsa_pack.cpp (the
// C ABI dispatch) and gqsa_pack_tc.cpp (product-internal).
#pragma once
#include <stddef.h>
#include <stdint.h>

#include "../../include/gqsa.h"
#include "gqsa_layout.h"

namespace gqsa {
int pack_tc_size(const gqsa_bsr_t* bsr, int32_t row_begin, int32_t row_end, size_t* blob_bytes);
int pack_tc(const gqsa_bsr_t* bsr, int32_t row_begin, int32_t row_end, void* blob, size_t blob_bytes,
            gqsa_desc_t* desc);
int read_desc_tc(const BlobHeader& h, const uint8_t* blob);
int unpack_tc(const gqsa_desc_t& d, const uint8_t* blob, gqsa_bsr_t* out);
}  // namespace gqsa
