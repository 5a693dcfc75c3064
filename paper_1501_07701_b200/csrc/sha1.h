// sha1.h -- minimal SHA-1 (FIPS 180-4) for characteristic-polynomial digests.
// The reference digests its charpolys with OpenSSL EVP SHA-1 (proj/src/dynamic_creator.cpp:11-34);
// MTGP parameter tables carry the SHA-1 of the polynomial printed as '0'/'1' coefficients,
// lowest degree first (verified against curand_mtgp32dc_p_11213.h).
#pragma once

#include <cstdint>
#include <string>

namespace mtgpb {
std::string sha1_hex(const std::string& data);
}  // namespace mtgpb
