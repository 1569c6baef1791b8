// b200_redirect.hpp -- the INTEGRATION.md binding, as a maintainer would add
// it: force-included (g++ -include) ahead of an UNMODIFIED reference source
// (proj/tests/acceptance/acceptance_main.cpp, proj/tests/test_ple.cpp), it
// pulls in the reference headers, then the B200 wrapper, then rebinds the
// reference's entry points so every call site in that source runs on the
// device. The reference's own inline code (parsed above the #defines) is not
// affected; only the calls the test makes are redirected.
//
//   block_iterative_ple  (ple.hpp:166)        -> gf2::b200::block_iterative_ple
//   recursive_ple        (ple.hpp:246)        -> gf2::b200::recursive_ple
//   rref_from_ple        (ple.hpp:318)        -> gf2::b200::rref_from_ple
//   echelonize           (m4ri.hpp:87)        -> gf2::b200::echelonize
//   partial_ple          (ple.hpp:57)         -> gf2::b200::partial_ple  (with GF2_B200_PARTIAL)
//   undo_column_swaps    (ple.hpp:293)        -> gf2::b200::undo_column_swaps (with GF2_B200_PARTIAL)
#pragma once

#include "gf2/gf2.hpp"
#include "gf2cu/ple.hpp"

#define block_iterative_ple(...) b200::block_iterative_ple(__VA_ARGS__)
#define recursive_ple(...) b200::recursive_ple(__VA_ARGS__)
#define rref_from_ple(...) b200::rref_from_ple(__VA_ARGS__)
#define echelonize(...) b200::echelonize(__VA_ARGS__)
#ifdef GF2_B200_PARTIAL
#define partial_ple(...) b200::partial_ple(__VA_ARGS__)
#define undo_column_swaps(...) b200::undo_column_swaps(__VA_ARGS__)
#endif
