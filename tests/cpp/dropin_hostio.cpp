// Host-side pieces of the drop-in (libspotlight_b200.so) driven from the
// command line, so tests/test_host_pins.py can compare them with the
// unmodified reference (oracle/_ref/libspotref.so) without a GPU:
// the initialisers (mlp_gaussian_init, qr_rotation_init, downproj_init,
// random_rotation) and the SPLH / SPLC file formats in both directions.
//
//   gauss d h L gamma seed out.bin        w1 | b1 | w2 as raw f32
//   qr d seed out.bin                     projection, raw f32
//   downproj d r seed out.bin             projection, raw f32
//   rotation d seed out.bin               random_rotation, raw f64
//   hasher_mlp d h L gamma seed out.splh  mlp_gaussian_init -> write_hasher
//   hasher_linear d seed out.splh         qr_rotation_init -> write_hasher
//   hasher_downproj d r seed out.splh     downproj_init -> write_hasher
//   rehasher in.splh out.splh             read_hasher -> write_hasher
//   codes_raw n L in.bin out.splc         raw u32 words -> write_code_index
//   recodes in.splc out.splc              read_code_index -> write_code_index
//   codes_dump in.splc out.bin            read_code_index -> raw u32 words
//   readhasher in.splh / readcodes in.splc   prints "ok" or "<Type>: <what()>"
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "spotlight/bitcodes.hpp"
#include "spotlight/errors.hpp"
#include "spotlight/hashers.hpp"
#include "spotlight/linalg.hpp"

using namespace spotlight;

namespace {

template <typename T>
void dump(const std::string& path, const T* p, size_t n) {
    std::ofstream f(path, std::ios::binary);
    f.write(reinterpret_cast<const char*>(p), sizeof(T) * n);
}

std::vector<char> slurp(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    return std::vector<char>(std::istreambuf_iterator<char>(f), {});
}

unsigned long long num(const char* s) { return std::strtoull(s, nullptr, 10); }

int run(int argc, char** argv) {
    const std::string cmd = argc > 1 ? argv[1] : "";
    if (cmd == "gauss" && argc == 8) {
        const MlpHasher m = mlp_gaussian_init(num(argv[2]), num(argv[3]), num(argv[4]),
                                              std::strtof(argv[5], nullptr), num(argv[6]));
        std::vector<float> all(m.w1.values());
        all.insert(all.end(), m.b1.begin(), m.b1.end());
        all.insert(all.end(), m.w2.values().begin(), m.w2.values().end());
        dump(argv[7], all.data(), all.size());
    } else if (cmd == "qr" && argc == 5) {
        const LinearHasher l = qr_rotation_init(num(argv[2]), num(argv[3]));
        dump(argv[4], l.projection.data(), l.projection.size());
    } else if (cmd == "downproj" && argc == 6) {
        const DownProjEstimator e = downproj_init(num(argv[2]), num(argv[3]), num(argv[4]));
        dump(argv[5], e.projection.data(), e.projection.size());
    } else if (cmd == "rotation" && argc == 5) {
        const Matrix<double> q = random_rotation(num(argv[2]), num(argv[3]));
        dump(argv[4], q.data(), q.size());
    } else if (cmd == "hasher_mlp" && argc == 8) {
        write_hasher(argv[7], AnyHasher{mlp_gaussian_init(num(argv[2]), num(argv[3]), num(argv[4]),
                                                          std::strtof(argv[5], nullptr),
                                                          num(argv[6]))});
    } else if (cmd == "hasher_linear" && argc == 5) {
        write_hasher(argv[4], AnyHasher{qr_rotation_init(num(argv[2]), num(argv[3]))});
    } else if (cmd == "hasher_downproj" && argc == 6) {
        write_hasher(argv[5], AnyHasher{downproj_init(num(argv[2]), num(argv[3]), num(argv[4]))});
    } else if (cmd == "rehasher" && argc == 4) {
        write_hasher(argv[3], read_hasher(argv[2]));
    } else if (cmd == "codes_raw" && argc == 6) {
        const std::vector<char> raw = slurp(argv[4]);
        CodeMatrix c(num(argv[2]), num(argv[3]));
        if (raw.size() != c.raw().size() * 4) {
            std::fprintf(stderr, "codes_raw: %zu bytes, want %zu\n", raw.size(), c.raw().size() * 4);
            return 2;
        }
        std::memcpy(c.raw().data(), raw.data(), raw.size());
        write_code_index(argv[5], c);
    } else if (cmd == "recodes" && argc == 4) {
        write_code_index(argv[3], read_code_index(argv[2]));
    } else if (cmd == "codes_dump" && argc == 4) {
        const CodeMatrix c = read_code_index(argv[2]);
        dump(argv[3], c.raw().data(), c.raw().size());
    } else if ((cmd == "readhasher" || cmd == "readcodes") && argc == 3) {
        try {
            if (cmd == "readhasher")
                (void)read_hasher(argv[2]);
            else
                (void)read_code_index(argv[2]);
            std::printf("ok\n");
        } catch (const FormatError& e) {
            std::printf("FormatError: %s\n", e.what());
        } catch (const IoError& e) {
            std::printf("IoError: %s\n", e.what());
        } catch (const DimensionError& e) {
            std::printf("DimensionError: %s\n", e.what());
        }
    } else {
        std::fprintf(stderr, "usage: see the header of tests/cpp/dropin_hostio.cpp\n");
        return 2;
    }
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        return run(argc, argv);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
