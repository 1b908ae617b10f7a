// kronbatch/kronbatch.hpp -- umbrella header of the drop-in API
// (reference: proj/include/kronbatch/kronbatch.hpp:1-9). The reference's
// brute-force oracle (reference.hpp) is test infrastructure and lives in
// oracle/, not in the product headers.
#pragma once

#include <kronbatch/types.hpp>
#include <kronbatch/views.hpp>
#include <kronbatch/kron1.hpp>
#include <kronbatch/kron2.hpp>
#include <kronbatch/kron3.hpp>
#include <kronbatch/gemm_a.hpp>
