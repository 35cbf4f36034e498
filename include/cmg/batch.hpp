// Drop-in forwarding header: the reference's include/cmg/batch.hpp (run_*_batch, time_run, bench_*) resolved
// to the B200 path. Put <repo>/include on the include path instead of the
// reference's; everything lives in cmgb_cmg.hpp.
#pragma once
#include "../cmgb_cmg.hpp"
