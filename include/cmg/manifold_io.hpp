// Drop-in forwarding header: the reference's include/cmg/manifold_io.hpp
// (write_manifold_csv, manifold_to_json) resolved to the B200 path. Put
// <repo>/include on the include path instead of the reference's; everything
// lives in cmgb_cmg.hpp.
#pragma once
#include "../cmgb_cmg.hpp"
