// frwcap/rng.hpp -- source-level drop-in for the reference header
// proj/include/frwcap/rng.hpp: the B200 build declares the whole frwcap API in
// one header (../frwcap.hpp), so callers of the reference that include
// "frwcap/rng.hpp" compile unchanged against it.
#pragma once
#include "../frwcap.hpp"
