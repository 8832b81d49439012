// frwcap/microwalk.hpp -- source-level drop-in for the reference header
// proj/include/frwcap/microwalk.hpp: the B200 build declares the whole frwcap API in
// one header (../frwcap.hpp), so callers of the reference that include
// "frwcap/microwalk.hpp" compile unchanged against it.
#pragma once
#include "../frwcap.hpp"
